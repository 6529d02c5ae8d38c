"""Vendor comparator: cuSPARSE 12.5 (the CUDA 12.9 toolkit's libcusparse)
fp64 CSR SpMV and CSR triangular solves (SpSV), called through its generic
API with ctypes -- descriptors, buffers and the SpSV analysis are built once,
so each timed call is the vendor kernel alone (the best case for it).

What it stands beside ("vendor comparator"):
  * SpMV y = L x on the canonical CSR (f64 values; int32 row offsets and
    columns, the one index type cuSPARSE takes for both below 2^31 nonzeros): the reference's spmv, /root/reference/pkg/src/lapeig/sparse.py:128-139,
    next to lg_spmv (wspmv_kernel).
  * z = (L L^T)^{-1} r as two SpSV calls on the IC(0) factor L (lower, non-unit
    diagonal; the second with op = TRANSPOSE): the reference's Ic0Factor.apply,
    ic0.py:40-45, next to lg_ic0_apply (sweep_flow_kernel).
Benchmark support only: nothing in the package imports this.
"""
import ctypes
import ctypes.util
import os

import numpy as np

_CUDA_R_64F = 1
_IDX32, _IDX64 = 2, 3
_BASE0 = 0
_NON_T, _T = 0, 1
_FILL, _DIAG = 0, 1          # cusparseSpMatAttribute_t
_LOWER, _NON_UNIT = 0, 0
SPMV_ALGS = {"default": 0, "csr_alg1": 2, "csr_alg2": 3}

_lib = None


def lib():
    global _lib
    if _lib is None:
        for cand in ("/usr/local/cuda/lib64/libcusparse.so.12", "libcusparse.so.12",
                     ctypes.util.find_library("cusparse")):
            if not cand:
                continue
            try:
                _lib = ctypes.CDLL(cand)
                break
            except OSError:
                continue
        if _lib is None:
            raise OSError("libcusparse.so.12 not found")
    return _lib


def _ck(rc, what):
    if rc != 0:
        raise RuntimeError(f"{what} failed: cusparseStatus {rc}")


class Handle:
    def __init__(self, stream_ptr=0):
        self.h = ctypes.c_void_p()
        _ck(lib().cusparseCreate(ctypes.byref(self.h)), "cusparseCreate")
        _ck(lib().cusparseSetStream(self.h, ctypes.c_void_p(stream_ptr)), "cusparseSetStream")


def _index_arrays(row_ptr, col_idx):
    """Row offsets and columns in ONE index type (cuSPARSE's generic CSR API
    rejects mixed 64/32-bit index types): int32 when nnz < 2^31, else int64."""
    import torch
    wide = int(row_ptr[-1]) >= 2**31 - 1
    dt = np.int64 if wide else np.int32
    rp = torch.from_numpy(np.asarray(row_ptr, dtype=dt)).cuda()
    col = torch.from_numpy(np.asarray(col_idx, dtype=dt)).cuda()
    return rp, col, (_IDX64 if wide else _IDX32)


def _csr(n, nnz, rp, col, val, idx):
    m = ctypes.c_void_p()
    _ck(lib().cusparseCreateCsr(ctypes.byref(m), ctypes.c_int64(n), ctypes.c_int64(n),
                                ctypes.c_int64(nnz), ctypes.c_void_p(rp.data_ptr()),
                                ctypes.c_void_p(col.data_ptr()), ctypes.c_void_p(val.data_ptr()),
                                idx, idx, _BASE0, _CUDA_R_64F), "cusparseCreateCsr")
    return m


def _dn(t):
    v = ctypes.c_void_p()
    _ck(lib().cusparseCreateDnVec(ctypes.byref(v), ctypes.c_int64(t.numel()),
                                  ctypes.c_void_p(t.data_ptr()), _CUDA_R_64F),
        "cusparseCreateDnVec")
    return v


class SpMV:
    """y = A x with cuSPARSE (A: host CSR arrays uploaded once)."""

    def __init__(self, handle, row_ptr, col_idx, values, x, y, alg="default"):
        import torch
        self.h = handle
        n = len(row_ptr) - 1
        self.rp, self.col, idx = _index_arrays(row_ptr, col_idx)
        self.val = torch.from_numpy(np.asarray(values, dtype=np.float64)).cuda()
        self.A = _csr(n, len(values), self.rp, self.col, self.val, idx)
        self.vx, self.vy = _dn(x), _dn(y)
        self.alg = SPMV_ALGS[alg]
        self.one, self.zero = ctypes.c_double(1.0), ctypes.c_double(0.0)
        size = ctypes.c_size_t()
        _ck(lib().cusparseSpMV_bufferSize(self.h.h, _NON_T, ctypes.byref(self.one), self.A,
                                          self.vx, ctypes.byref(self.zero), self.vy,
                                          _CUDA_R_64F, self.alg, ctypes.byref(size)),
            "cusparseSpMV_bufferSize")
        self.buf = torch.empty(max(size.value, 16), dtype=torch.uint8, device="cuda")
        _ck(lib().cusparseSpMV_preprocess(self.h.h, _NON_T, ctypes.byref(self.one), self.A,
                                          self.vx, ctypes.byref(self.zero), self.vy,
                                          _CUDA_R_64F, self.alg,
                                          ctypes.c_void_p(self.buf.data_ptr())),
            "cusparseSpMV_preprocess")

    def __call__(self):
        _ck(lib().cusparseSpMV(self.h.h, _NON_T, ctypes.byref(self.one), self.A, self.vx,
                               ctypes.byref(self.zero), self.vy, _CUDA_R_64F, self.alg,
                               ctypes.c_void_p(self.buf.data_ptr())), "cusparseSpMV")


class Ic0Apply:
    """z = (L L^T)^{-1} r: SpSV with L, then SpSV with L^T (op = TRANSPOSE)
    on the same lower CSR factor; analysis once per direction."""

    def __init__(self, handle, row_ptr, col_idx, values, r, z):
        import torch
        self.h = handle
        n = len(row_ptr) - 1
        self.rp, self.col, idx = _index_arrays(row_ptr, col_idx)
        self.val = torch.from_numpy(np.asarray(values, dtype=np.float64)).cuda()
        self.L = _csr(n, len(values), self.rp, self.col, self.val, idx)
        fill, diag = ctypes.c_int(_LOWER), ctypes.c_int(_NON_UNIT)
        _ck(lib().cusparseSpMatSetAttribute(self.L, _FILL, ctypes.byref(fill), 4), "fill")
        _ck(lib().cusparseSpMatSetAttribute(self.L, _DIAG, ctypes.byref(diag), 4), "diag")
        self.w = torch.empty(n, dtype=torch.float64, device="cuda")
        self.vr, self.vw, self.vz = _dn(r), _dn(self.w), _dn(z)
        self.one = ctypes.c_double(1.0)
        self.steps = []
        for op, vin, vout in ((_NON_T, self.vr, self.vw), (_T, self.vw, self.vz)):
            d = ctypes.c_void_p()
            _ck(lib().cusparseSpSV_createDescr(ctypes.byref(d)), "cusparseSpSV_createDescr")
            size = ctypes.c_size_t()
            _ck(lib().cusparseSpSV_bufferSize(self.h.h, op, ctypes.byref(self.one), self.L, vin,
                                              vout, _CUDA_R_64F, 0, d, ctypes.byref(size)),
                "cusparseSpSV_bufferSize")
            buf = torch.empty(max(size.value, 16), dtype=torch.uint8, device="cuda")
            _ck(lib().cusparseSpSV_analysis(self.h.h, op, ctypes.byref(self.one), self.L, vin,
                                            vout, _CUDA_R_64F, 0, d,
                                            ctypes.c_void_p(buf.data_ptr())),
                "cusparseSpSV_analysis")
            self.steps.append((op, vin, vout, d, buf))

    def __call__(self):
        for op, vin, vout, d, _ in self.steps:
            _ck(lib().cusparseSpSV_solve(self.h.h, op, ctypes.byref(self.one), self.L, vin, vout,
                                         _CUDA_R_64F, 0, d), "cusparseSpSV_solve")


def vendor_block(a, f, x_dev, timer, flush=None):
    """cuSPARSE SpMV (every algorithm) and the IC(0) apply as two SpSVs on
    matrix `a` / factor `f` (reference CsrMatrix / Ic0Factor), each timed by
    `timer(fn)` (microseconds) and checked against the package's products."""
    import torch
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev
    h = Handle(torch.cuda.current_stream().cuda_stream)
    out = {"library": f"cuSPARSE (libcusparse {os.path.basename(lib()._name)})",
           "spmv": {}, "format": "CSR int32 row offsets and columns (int64 when nnz >= 2^31), f64 values"}
    d = a.device()
    y_ours = dev.empty(a.n)
    d.matvec(x_dev, y_ours)
    for alg in SPMV_ALGS:
        y = torch.empty(a.n, dtype=torch.float64, device="cuda")
        try:
            op = SpMV(h, a.row_ptr, a.col_idx, a.values, x_dev, y, alg)
            op()
            torch.cuda.synchronize()
            err = float((y - y_ours).abs().max() / y_ours.abs().max())
            out["spmv"][alg] = {"us": timer(op, flush), "max_rel_diff_vs_lg_spmv": err}
        except Exception as ex:  # noqa: BLE001 - report, do not fail the bench
            out["spmv"][alg] = {"error": repr(ex)[:200]}
    out["lg_spmv_us"] = timer(lambda: d.matvec(x_dev, y_ours), flush)
    if f is not None:
        fl = f.l
        z = torch.empty(a.n, dtype=torch.float64, device="cuda")
        try:
            op = Ic0Apply(h, fl.row_ptr, fl.col_idx, fl.values, x_dev, z)
            op()
            fd = f.device()
            z_ours = dev.empty(a.n)
            fd.apply(x_dev, z_ours)
            torch.cuda.synchronize()
            err = float((z - z_ours).abs().max() / z_ours.abs().max())
            out["ic0_apply_spsv"] = {"us": timer(op, flush), "max_rel_diff_vs_lg_ic0_apply": err,
                                     "calls": "SpSV(L) then SpSV(L^T), analysis outside the timing"}
            out["lg_ic0_apply_us"] = timer(lambda: fd.apply(x_dev, z_ours), flush)
        except Exception as ex:  # noqa: BLE001
            out["ic0_apply_spsv"] = {"error": repr(ex)[:200]}
    return out
