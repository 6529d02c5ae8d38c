"""ctypes binding of liblapb200.so (include/lapb200.h).

This module is the only place that touches the C ABI.  It loads the in-tree
library, declares every entry point, mirrors the argument structs, and maps
status codes onto the reference's exception types:

    LG_EINVAL     -> ValueError      (sparse.py:131-132, dacg.py:138-143, ...)
    LG_EBREAKDOWN -> ic0.Ic0Error     (ic0.py:20)
    anything else -> RuntimeError

There is deliberately no fallback: if the library is missing or no CUDA
device is visible, every hot-path call raises.
"""

import ctypes
import os
import threading
from pathlib import Path

LIB_PATH = Path(__file__).resolve().parent / "_lib" / "liblapb200.so"

LG_OK = 0
LG_EINVAL = -1
LG_ECUDA = -2
LG_ENOMEM = -3
LG_EBREAKDOWN = -4
LG_EFORMAT = -5

LG_CSR_PLAIN = 1
LG_CSR_SKIP_EMPTY = 2
LG_MAXT = 4
LG_MAXD = 8
LG_MAXB = 2
LG_MAXO = 3
LG_MAXQ = 64
LG_MAXOPS = 192
LG_MAXIMM = 32

# sentinel operand pointers naming the outputs of the same fused pass
OUT0 = 1
OUT1 = 2
OUT2 = 3

c_p = ctypes.c_void_p
c_i64 = ctypes.c_int64
c_int = ctypes.c_int
c_dbl = ctypes.c_double


class Term(ctypes.Structure):
    _fields_ = [("v", c_p), ("h", c_dbl), ("d", c_p)]


class Output(ctypes.Structure):
    _fields_ = [
        ("out", c_p), ("nterms", c_int), ("t", Term * LG_MAXT),
        ("uq", c_p), ("uld", c_i64), ("uk", c_int), ("uc", c_p),
        ("cscale", c_dbl), ("uq2", c_p), ("uld2", c_i64), ("uk2", c_int), ("uc2", c_p),
        ("d_post", c_p), ("post_mode", c_int),
    ]


class Block(ctypes.Structure):
    _fields_ = [("q", c_p), ("ld", c_i64), ("k", c_int), ("v", c_p)]


class FusedArgs(ctypes.Structure):
    _fields_ = [
        ("n", c_i64), ("o", Output * LG_MAXO), ("ndots", c_int),
        ("da", c_p * LG_MAXD), ("db", c_p * LG_MAXD), ("dc", c_p * LG_MAXD),
        ("nblocks", c_int), ("b", Block * LG_MAXB),
        ("result", c_p), ("skip", c_p),
    ]


_SIGS = {
    "lg_last_error": (ctypes.c_char_p, []),
    "lg_version": (c_int, []),
    "lg_device_info": (c_int, [c_p, c_p, c_p, c_p]),
    "lg_readback": (c_int, [c_p, c_p, c_i64, c_p]),
    "lg_upload": (c_int, [c_p, c_p, c_i64, c_p]),
    "lg_capture_begin": (c_int, [c_p]),
    "lg_capture_end": (c_int, [c_p, c_p]),
    "lg_graph_launch": (c_int, [c_p, c_p]),
    "lg_graph_destroy": (c_int, [c_p]),
    "lg_ws_create": (c_int, [c_p]),
    "lg_ws_destroy": (c_int, [c_p]),
    "lg_csr_create": (c_int, [c_i64, c_i64, c_p, c_p, c_p, c_int, c_p]),
    "lg_csr_destroy": (c_int, [c_p]),
    "lg_csr_info": (c_int, [c_p, c_p, c_p, c_p, c_p, c_p, c_p]),
    "lg_csr_download": (c_int, [c_p, c_p, c_p, c_p]),
    "lg_spmv": (c_int, [c_p, c_p, c_p, c_dbl, c_p, c_int, c_int, c_p, c_p,
                        c_i64, c_int, c_p, c_p, c_p, c_p]),
    "lg_spmv_gather_probe": (c_int, [c_p, c_p, c_p, c_p]),
    "lg_spmv_host": (c_int, [c_p, c_p, c_p, c_p, c_p, c_p]),
    "lg_spmm": (c_int, [c_p, c_p, c_p, c_int, c_p]),
    "lg_spmm_rowmajor": (c_int, [c_p, c_p, c_p, c_int, c_p, c_p]),
    "lg_rmat_device": (c_int, [c_int, c_int, c_dbl, c_dbl, c_dbl, ctypes.c_uint64, c_p, c_p,
                               c_p]),
    "lg_lcc_device": (c_int, [c_i64, c_i64, c_p, c_p, c_p, c_p]),
    "lg_csr_laplacian_device": (c_int, [c_i64, c_i64, c_p, c_p, c_p]),
    "lg_csr_diagonal": (c_int, [c_p, c_p]),
    "lg_free": (c_int, [c_p]),
    "lg_build_laplacian": (c_int, [c_i64, c_i64, c_p, c_p, c_p, c_p, c_p, c_p]),
    "lg_ic0_factorize": (c_int, [c_i64, c_p, c_p, c_p, c_dbl, c_p, c_int, c_p,
                                 c_p, c_p, c_p, c_p]),
    "lg_ic0_create": (c_int, [c_i64, c_p, c_p, c_p, c_p]),
    "lg_ic0_create_perm": (c_int, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "lg_ic0_destroy": (c_int, [c_p]),
    "lg_color_smallest_last": (c_int, [c_i64, c_p, c_p, c_p, c_p]),
    "lg_ic0_info": (c_int, [c_p, c_p, c_p, c_p]),
    "lg_ic0_apply": (c_int, [c_p, c_p, c_p, c_p, c_p]),
    "lg_ic0_set_mode": (c_int, [c_p, c_int]),
    "lg_ic0_sweep_depth": (c_int, [c_p, c_p, c_p, c_p]),
    "lg_ic0_merged_solve_host": (c_int, [c_i64, c_p, c_p, c_p, c_int, c_int, c_p, c_p, c_p, c_p,
                                         c_p]),
    "lg_ic0_trace": (c_int, [c_p, c_int, c_p, c_int]),
    "lg_ic0_flow_trace": (c_int, [c_p, c_int, c_p, c_int]),
    "lg_ic0_schedule": (c_int, [c_p, c_int, c_p, c_int]),
    "lg_diag_apply": (c_int, [c_i64, c_p, c_p, c_p, c_p, c_p]),
    "lg_fused": (c_int, [c_p, c_p, c_p]),
    "lg_csr_row_block": (c_int, [c_p, c_i64, c_i64, c_p]),
    "lg_csr_row_ptr": (c_int, [c_p, c_p]),
    "lg_csr_export_host": (c_int, [c_p, c_p, c_p, c_p]),
    "lg_csr_split_cols": (c_int, [c_p, c_i64, c_i64, c_p, c_p]),
    "lg_csr_col_panel": (c_int, [c_p, c_i64, c_i64, c_int, c_p]),
    "lg_csr_set_panels": (c_int, [c_p, c_int]),
    "lg_fsai_nnz": (c_int, [c_i64, c_p, c_p, c_p, c_int, c_int, c_p]),
    "lg_graph_parse": (c_int, [c_p, c_i64, c_int, c_int, c_p, c_p, c_p, c_p, c_p, c_p]),
    "lg_host_free": (c_int, [c_p]),
    "lg_fsai_factorize": (c_int, [c_i64, c_p, c_p, c_p, c_int, c_int, c_p, c_p, c_p]),
    "lg_fsai_device": (c_int, [c_p, c_int, c_p, c_p]),
    "lg_spmv_acc": (c_int, [c_p, c_p, c_p, c_p, c_p, c_p]),
    "lg_fused_prog": (c_int, [c_p, c_p, c_p, c_p, c_int, c_p, c_int, c_p, c_p]),
    "lg_gemm_small": (c_int, [c_i64, c_p, c_i64, c_int, c_p, c_int, c_p, c_i64, c_p]),
    "lg_scalar_prog": (c_int, [c_p, c_p, c_p, c_int, c_p, c_int, c_p, c_p]),
}

EXPORTED = tuple(sorted(_SIGS))

_lock = threading.Lock()
_lib = None


def load():
    """The loaded library (raises if it was not built)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not LIB_PATH.exists():
                raise RuntimeError(
                    f"{LIB_PATH} is missing: build it with "
                    "`python -m paper_1311_1695_b200.build` (there is no CPU fallback)")
            # LG_LIB_OVERRIDE: an alternative build of the same library
            # (A/B timing of kernel variants in one process tree; dev only)
            path = os.environ.get("LG_LIB_OVERRIDE") or str(LIB_PATH)
            lib = ctypes.CDLL(path)
            for name, (res, args) in _SIGS.items():
                if os.environ.get("LG_LIB_OVERRIDE") and not hasattr(lib, name):
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def last_error():
    return load().lg_last_error().decode(errors="replace")


def check(rc, what=""):
    """Raise the reference-style exception for a nonzero status."""
    if rc == LG_OK:
        return
    msg = last_error()
    if what:
        msg = f"{what}: {msg}"
    if rc == LG_EINVAL:
        raise ValueError(msg)
    if rc == LG_EBREAKDOWN:
        from .ic0 import Ic0Error
        raise Ic0Error(msg)
    raise RuntimeError(msg)


def call(name, *args):
    check(getattr(load(), name)(*args), name)
