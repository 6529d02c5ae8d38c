"""Device preconditioners behind the reference's preconditioner seam.

The reference accepts None, a callable, or any object with .apply(r)
(pcg.py:112-117, dacg.py:187).  The device solvers need an object with
apply_raw(r_ptr, z_ptr, skip, stream); device_preconditioner() adapts:

    Ic0Factor (this package or the reference's)  -> DeviceIc0 sweeps
    JacobiFactor (flagged, non-reference variant) -> diagonal scaling
    None                                          -> identity (a copy)
    any other object with .apply / callable       -> called on CUDA tensors
"""

import weakref

import numpy as np

from . import _device as dev
from . import _native as nat
from ._plan import Fused

_cache = weakref.WeakKeyDictionary()


class IdentityPrec:
    def __init__(self, n):
        self.n = n

    def apply_raw(self, r, z, skip, stream):
        a = nat.FusedArgs()
        a.n = self.n
        a.o[0].out = z
        a.o[0].nterms = 1
        a.o[0].t[0].v = r
        a.o[0].t[0].h = 1.0
        a.skip = skip
        nat.check(nat.load().lg_fused(ctypes_byref(a), dev.workspace().handle, stream), "copy")

    def apply(self, r, z=None):
        z = dev.empty(self.n) if z is None else z
        Fused(self.n, outs=[dict(out=z, terms=[(r, 1.0)])])()
        return z


def ctypes_byref(a):
    import ctypes
    return ctypes.byref(a)


class JacobiFactor:
    """Diagonal (Jacobi) preconditioner, z = r / diag(A).

    A flagged NON-reference variant: no triangular solve, at
    1.8-3.8x the reference's MVP counts.  Same .apply seam as Ic0Factor.
    """

    def __init__(self, a):
        d = np.asarray(a.diagonal(), dtype=np.float64)
        if np.any(d <= 0):
            raise ValueError("Jacobi preconditioner needs a positive diagonal")
        self.n = int(a.n)
        self.shift = 0.0
        self.attempts = 0
        self._dinv = dev.to_device(1.0 / d)

    def apply_raw(self, r, z, skip, stream):
        nat.check(nat.load().lg_diag_apply(self.n, self._dinv.data_ptr(), r, z, skip, stream),
                  "lg_diag_apply")

    def device(self):
        return self

    def apply(self, r, z=None):
        on_dev = dev.is_device_array(r)
        rd = dev.to_device(r)
        out = dev.empty(self.n) if z is None else z
        self.apply_raw(rd.data_ptr(), out.data_ptr(), None, dev.stream_ptr())
        return out if on_dev else dev.to_host(out)


class FsaiFactor:
    """Factorized sparse approximate inverse, z = G^T G r (lg_fsai.cu).

    A flagged NON-reference variant: the approximate inverse the paper
    proposes as the parallel-friendly alternative (SURVEY
    8(f) item 3).  G is lower triangular on the lower pattern of A with at
    most kmax entries per row (hub rows keep their kmax - 1 largest |a_ij|);
    the apply is two SpMVs -- no triangular dependency chain, and across GPUs
    two row-partitioned SpMVs without the block-Jacobi loss.  Same .apply
    seam as Ic0Factor.  Scratch is per thread, so a factor can be shared by
    solves on different threads.
    """

    def __init__(self, a, kmax=32, levels=1):
        import ctypes

        from .sparse import CsrMatrix, DeviceCsr
        n = int(a.n)
        rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
        col = np.ascontiguousarray(a.col_idx, dtype=np.int64)
        val = np.ascontiguousarray(a.values, dtype=np.float64)
        nnz = ctypes.c_int64()
        nat.call("lg_fsai_nnz", n, rp.ctypes.data, col.ctypes.data if col.size else None,
                 val.ctypes.data if val.size else None, int(kmax), int(levels),
                 ctypes.byref(nnz))
        grp = np.zeros(n + 1, dtype=np.int64)
        gcol = np.zeros(max(nnz.value, 1), dtype=np.int64)
        gval = np.zeros(max(nnz.value, 1), dtype=np.float64)
        nat.call("lg_fsai_factorize", n, rp.ctypes.data, col.ctypes.data if col.size else None,
                 val.ctypes.data if val.size else None, int(kmax), int(levels), grp.ctypes.data,
                 gcol.ctypes.data, gval.ctypes.data)
        gcol, gval = gcol[:nnz.value], gval[:nnz.value]
        self.n = n
        self.kmax = int(kmax)
        self.levels = int(levels)
        self.shift = 0.0
        self.attempts = 0
        self.g = CsrMatrix(n, grp, gcol, gval)
        # G^T by a stable sort on the column index (rows of G ascending)
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(grp))
        order = np.argsort(gcol, kind="stable")
        trp = np.zeros(n + 1, dtype=np.int64)
        np.add.at(trp, gcol + 1, 1)
        self.gt = CsrMatrix(n, np.cumsum(trp), rows[order], gval[order])
        self._dg = self._dgt = self._tmp = None
        self._dev_ready = False
        self._DeviceCsr = DeviceCsr

    @classmethod
    def from_device(cls, a, kmax=32):
        """The FSAI of a device-only packed matrix with one off-diagonal
        value (a unit-weight Laplacian such as rmat_laplacian_device's),
        built on the device (lg_fsai_device).  Single-GPU only (no host
        copy of G for row-partitioned solves)."""
        import ctypes

        from .sparse import DeviceCsr
        d = a.device()
        hg, hgt = ctypes.c_void_p(), ctypes.c_void_p()
        nat.call("lg_fsai_device", d.handle, int(kmax), ctypes.byref(hg), ctypes.byref(hgt))
        self = cls.__new__(cls)
        self.n = int(a.n)
        self.kmax = int(kmax)
        self.shift = 0.0
        self.attempts = 0
        self.g = self.gt = None
        self._DeviceCsr = DeviceCsr
        info = [ctypes.c_int64() for _ in range(4)] + [ctypes.c_int(), ctypes.c_int64()]
        nat.call("lg_csr_info", hg, *[ctypes.byref(v) for v in info])
        self._dg = DeviceCsr.from_handle(hg, self.n, info[1].value)
        self._dgt = DeviceCsr.from_handle(hgt, self.n, info[1].value)
        self._tmp = dev.empty(self.n)
        self._dev_ready = True
        return self

    def _ensure(self):
        if not self._dev_ready:
            self._dg = self._DeviceCsr(self.n, self.g.row_ptr, self.g.col_idx, self.g.values)
            self._dgt = self._DeviceCsr(self.n, self.gt.row_ptr, self.gt.col_idx,
                                        self.gt.values)
            self._tmp = dev.empty(self.n)
            self._dev_ready = True

    def _scratch(self):
        """G r of the apply: one scratch vector per thread, so solves on
        different threads (streams) can share the factor."""
        import threading
        tls = self.__dict__.setdefault("_tls", threading.local())
        t = getattr(tls, "t", None)
        if t is None:
            t = tls.t = dev.empty(self.n)
        return t

    def apply_raw(self, r, z, skip, stream):
        self._ensure()
        ws = dev.workspace().handle
        lib = nat.load()
        tmp = self._scratch().data_ptr()
        for m, src, dst in ((self._dg, r, tmp), (self._dgt, tmp, z)):
            nat.check(lib.lg_spmv(m.handle, src, dst, 0.0, None, 0, 0, None, None, 0, 0, None,
                                  ws, skip, stream), "lg_spmv")

    def device(self):
        self._ensure()
        return self

    def apply(self, r, z=None):
        on_dev = dev.is_device_array(r)
        rd = dev.to_device(r)
        if tuple(rd.shape) != (self.n,):
            raise ValueError("vector length does not match factor dimension")
        out = dev.empty(self.n) if z is None else z
        self.apply_raw(rd.data_ptr(), out.data_ptr(), None, dev.stream_ptr())
        return out if on_dev else dev.to_host(out)


def fsai_factorize(a, kmax=32, levels=1):
    """FSAI preconditioner of a (flagged non-reference variant); levels=2
    widens each row's pattern to second-level neighbours (FSAI(2))."""
    return FsaiFactor(a, kmax, levels)


class Ic0JacobiFactor:
    """IC(0) with its triangular solves replaced by s Jacobi sweeps each
    (flagged NON-reference variant: "Jacobi-sweep
    approximate triangular solves").

    With L = D + N the reference's IC(0) factor (ic0.py:48-116, D its
    diagonal), L^{-1} = sum_i (-D^{-1} N)^i D^{-1} (N D^{-1} nilpotent), and
    s sweeps y <- D^{-1} r - D^{-1} N y from y = D^{-1} r keep the first
    s + 1 terms, G_s.  The backward sweeps on L^T keep exactly the terms of
    G_s^T, so z = G_s^T G_s r: symmetric positive definite for every s, and
    the exact IC(0) apply once s reaches the factor's level count.  Each
    sweep is two launches: y' = D^{-1} r (a diagonal lg_spmv) and y' += B y
    (lg_spmv_acc, B = -D^{-1} N or -D^{-1} N^T): no dependency chain, about
    (s + 1) half-Laplacian products per triangle.  Same .apply seam.
    """

    def __init__(self, f, sweeps=2):
        from .sparse import DeviceCsr
        l = f.l if hasattr(f, "l") else f
        sweeps = int(sweeps)
        if sweeps < 0:
            raise ValueError("sweeps must be >= 0")
        n = int(l.n)
        rp = np.asarray(l.row_ptr, dtype=np.int64)
        col = np.asarray(l.col_idx, dtype=np.int64)
        val = np.asarray(l.values, dtype=np.float64)
        rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
        on_diag = col == rows
        if np.count_nonzero(on_diag) != n:
            raise ValueError("factor needs a stored diagonal in every row")
        d = np.empty(n)
        d[rows[on_diag]] = val[on_diag]
        off = ~on_diag
        if np.any(col[off] > rows[off]):
            raise ValueError("factor must be lower triangular")
        orow, ocol = rows[off], col[off]
        bval = -val[off] / d[orow]                     # -D^{-1} N, row-scaled
        frp = np.zeros(n + 1, dtype=np.int64)
        np.add.at(frp, orow + 1, 1)
        frp = np.cumsum(frp)
        # -D^{-1} N^T: entry (j, i) = -n_ij / d_j, rows of N^T by a stable sort
        order = np.argsort(ocol, kind="stable")
        brp = np.zeros(n + 1, dtype=np.int64)
        np.add.at(brp, ocol + 1, 1)
        brp = np.cumsum(brp)
        tval = -val[off][order] / d[ocol[order]]
        self.n = n
        self.sweeps = sweeps
        self.shift = getattr(f, "shift", 0.0)
        self.attempts = getattr(f, "attempts", 0)
        from types import SimpleNamespace as _M
        idx = np.arange(n + 1, dtype=np.int64)
        # host triples (row-partitioned solves cut their row blocks from these)
        self.dinv = _M(n=n, row_ptr=idx, col_idx=np.arange(n, dtype=np.int64), values=1.0 / d)
        self.bf = _M(n=n, row_ptr=frp, col_idx=ocol, values=bval)
        self.bb = _M(n=n, row_ptr=brp, col_idx=orow[order], values=tval)
        self._dinv, self._bf, self._bb = (DeviceCsr(n, m.row_ptr, m.col_idx, m.values)
                                          for m in (self.dinv, self.bf, self.bb))

    def _scratch(self):
        import threading
        tls = self.__dict__.setdefault("_tls", threading.local())
        t = getattr(tls, "t", None)
        if t is None:
            t = tls.t = [dev.empty(self.n) for _ in range(3)]
        return t

    def apply_raw(self, r, z, skip, stream):
        ws = dev.workspace().handle
        lib = nat.load()
        t1, t2, p = [t.data_ptr() for t in self._scratch()]
        s = self.sweeps

        def diag(src, dst):
            nat.check(lib.lg_spmv(self._dinv.handle, src, dst, 0.0, None, 0, 0, None, None, 0,
                                  0, None, ws, skip, stream), "lg_spmv")

        def acc(m, src, dst):
            nat.check(lib.lg_spmv_acc(m.handle, src, dst, ws, skip, stream), "lg_spmv_acc")

        # forward: y_0 = D^-1 r, y_i = D^-1 r + B_f y_{i-1}   (t1 / t2)
        fw = [t1, t2]
        diag(r, fw[0])
        for i in range(1, s + 1):
            diag(r, fw[i % 2])
            acc(self._bf, fw[(i - 1) % 2], fw[i % 2])
        y = fw[s % 2]
        # backward on L^T, the last write landing in z   (z / p)
        bw = lambda i: z if (s - i) % 2 == 0 else p       # noqa: E731
        diag(y, bw(0))
        for i in range(1, s + 1):
            diag(y, bw(i))
            acc(self._bb, bw(i - 1), bw(i))

    def device(self):
        return self

    def apply(self, r, z=None):
        on_dev = dev.is_device_array(r)
        rd = dev.to_device(r)
        if tuple(rd.shape) != (self.n,):
            raise ValueError("vector length does not match factor dimension")
        out = dev.empty(self.n) if z is None else z
        self.apply_raw(rd.data_ptr(), out.data_ptr(), None, dev.stream_ptr())
        return out if on_dev else dev.to_host(out)


def ic0_jacobi_sweeps(f, sweeps=2):
    """IC(0) factor f (or its L) applied by `sweeps` Jacobi sweeps per
    triangle (flagged non-reference variant)."""
    return Ic0JacobiFactor(f, sweeps)


class CallablePrec:
    """Wraps a user callable / object with .apply (not graph-capturable)."""

    def __init__(self, fn, n):
        self.fn = fn
        self.n = n

    def apply_raw(self, r, z, skip, stream):
        raise RuntimeError("a Python-callable preconditioner cannot run inside a device plan")

    def apply(self, r, z=None):
        out = self.fn(r)
        out = out if dev.is_device_array(out) else dev.to_device(out)
        if z is None:
            return out
        z.copy_(out)
        return z


def device_preconditioner(f, n):
    """Device preconditioner for the solver seam `f`."""
    from .ic0 import DeviceIc0, Ic0Factor, MulticolorIc0Factor
    if f is None:
        return IdentityPrec(n)
    if isinstance(f, (Ic0Factor, MulticolorIc0Factor)):
        return f.device()
    if isinstance(f, (JacobiFactor, FsaiFactor, Ic0JacobiFactor)):
        return f.device()
    if hasattr(f, "l") and hasattr(f.l, "row_ptr"):
        # a foreign Ic0Factor-like object (the reference's own, ic0.py:24-45):
        # its device copy lives as long as the object, never longer
        try:
            hit = _cache.get(f)
            if hit is None:
                hit = _cache[f] = DeviceIc0(f.l)
            return hit
        except TypeError:   # not weak-referenceable: no caching
            return DeviceIc0(f.l)
    fn = f if callable(f) else f.apply
    return CallablePrec(fn, n)
