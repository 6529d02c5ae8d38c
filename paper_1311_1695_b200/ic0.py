"""No-fill incomplete Cholesky preconditioning on the B200.

Mirrors the reference module ic0.py (lapeig 0.1.0):

    SHIFT_SCHEDULE, Ic0Error                 ic0.py:16-21
    Ic0Factor(l, shift, attempts).apply(r)   ic0.py:24-45   z = (L L^T)^{-1} r
    ic0_factorize(a, shift0, schedule)       ic0.py:81-116  (host C++, bit-exact)
    identity_factor, precond_apply,
    projected_precond_apply                  ic0.py:134-150

The factorization runs once per matrix in liblapb200's host C++ (same
operation order as the reference, no FMA contraction: the factor is
identical bit for bit).  The apply is the device's two sync-free
triangular sweeps (csrc/lg_ic0.cu).  `Ic0Factor.apply` accepts numpy
(round trip through the device) or a CUDA tensor (stays on the device).
"""

import ctypes

import numpy as np

from . import _device as dev
from . import _native as nat
from .sparse import CsrMatrix

# retry shifts, tried in order until the factorization completes (ic0.py:16)
SHIFT_SCHEDULE = (1e-8, 1e-6, 1e-4, 1e-3, 1e-2)
_PIVOT_FLOOR = 1e-14


class Ic0Error(RuntimeError):
    """Factorization failed at every shift in the schedule."""


class DeviceIc0:
    """Device copy of a lower factor (an lg_ic0 handle) + sweep scratch.

    perm (optional): original row of every factor row, for the factor of a
    reordered matrix P A P^T; the apply then works in the original numbering.
    """

    def __init__(self, l, perm=None):
        dev.require_cuda()
        rp = np.ascontiguousarray(l.row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(l.col_idx, dtype=np.int64)
        va = np.ascontiguousarray(l.values, dtype=np.float64)
        h = ctypes.c_void_p()
        pm = None if perm is None else np.ascontiguousarray(perm, dtype=np.int64)
        nat.call("lg_ic0_create_perm", int(l.n), rp.ctypes.data,
                 ci.ctypes.data if ci.size else None, va.ctypes.data if va.size else None,
                 pm.ctypes.data if pm is not None else None, ctypes.byref(h))
        self.handle = h
        self.n = int(l.n)
        n_ = ctypes.c_int64()
        nnz = ctypes.c_int64()
        lev = ctypes.c_int()
        nat.call("lg_ic0_info", h, ctypes.byref(n_), ctypes.byref(nnz), ctypes.byref(lev))
        self.nnz_l = nnz.value
        self.levels = lev.value
        fw, bw, ent = ctypes.c_int(), ctypes.c_int(), ctypes.c_int64()
        nat.call("lg_ic0_sweep_depth", h, ctypes.byref(fw), ctypes.byref(bw), ctypes.byref(ent))
        # depth and entries of the sweeps as scheduled (level-merged form)
        self.sweep_levels = (fw.value, bw.value)
        self.sweep_entries = ent.value
        # algorithmic bytes of one apply: two sweeps over L
        # (f64 val + int32 col + int64 row_ptr) plus r, y, z traffic
        self.algo_bytes = 2 * (12 * self.nnz_l + 8 * (self.n + 1)) + 32 * self.n

    def __del__(self):
        h = getattr(self, "handle", None)
        if h and h.value and nat._lib is not None:
            nat._lib.lg_ic0_destroy(h)

    def set_mode(self, mode):
        """Sweep implementation: 0 dataflow sweeps (default), 1 resident
        one-CTA sweep (opt-in; same bits either way); -1 only queries.
        Returns the previous mode."""
        return nat.load().lg_ic0_set_mode(self.handle, int(mode))

    def apply_raw(self, r, z, skip, stream):
        nat.check(nat.load().lg_ic0_apply(self.handle, r, z, skip, stream), "lg_ic0_apply")

    def apply(self, r, z=None):
        """z = (L L^T)^{-1} r on device tensors."""
        if z is None:
            z = dev.empty(self.n)
        if self.n:
            self.apply_raw(r.data_ptr(), z.data_ptr(), None, dev.stream_ptr())
        return z


class Ic0Factor:
    """Lower-triangular incomplete Cholesky factor with its metadata.

    apply(r) solves (L L^T) z = r through two triangular solves.
    """

    __slots__ = ("l", "shift", "attempts", "_dev")

    def __init__(self, l, shift, attempts):
        self.l = l
        self.shift = float(shift)
        self.attempts = int(attempts)
        self._dev = None

    def device(self):
        if self._dev is None:
            self._dev = DeviceIc0(self.l)
        return self._dev

    def apply(self, r):
        on_dev = dev.is_device_array(r)
        shape = tuple(r.shape) if on_dev else np.asarray(r).shape
        if shape != (self.l.n,):
            raise ValueError("vector length does not match factor dimension")
        z = self.device().apply(dev.to_device(r))
        return z if on_dev else dev.to_host(z)


def ic0_factorize(a, shift0=0.0, schedule=SHIFT_SCHEDULE):
    """Incomplete Cholesky of a + alpha * diag(a) on the pattern of a.

    Tries alpha = shift0 first, then walks the schedule, finishing with
    0.1 * max diagonal entry as a last resort (ic0.py:81-116).  Raises
    Ic0Error when every shift fails.
    """
    if not a.symmetric:
        raise ValueError("incomplete Cholesky needs a symmetric matrix")
    n = int(a.n)
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
    va = np.ascontiguousarray(a.values, dtype=np.float64)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    nl = int(np.count_nonzero(ci < rows)) + n
    l_rp = np.empty(n + 1, dtype=np.int64)
    l_col = np.empty(max(nl, 1), dtype=np.int64)
    l_val = np.empty(max(nl, 1), dtype=np.float64)
    sched = np.ascontiguousarray(schedule, dtype=np.float64)
    shift = ctypes.c_double()
    attempts = ctypes.c_int()
    rc = nat.load().lg_ic0_factorize(
        n, rp.ctypes.data, ci.ctypes.data if ci.size else None,
        va.ctypes.data if va.size else None, float(shift0),
        sched.ctypes.data if sched.size else None, int(sched.size),
        l_rp.ctypes.data, l_col.ctypes.data, l_val.ctypes.data,
        ctypes.byref(shift), ctypes.byref(attempts))
    if rc == nat.LG_EBREAKDOWN:
        diag = a.diagonal()
        dmax = float(diag.max()) if n else 0.0
        shifts = [float(shift0)] + [s for s in schedule if s > shift0]
        last = 0.1 * dmax
        if dmax > 0 and (not shifts or last > shifts[-1]):
            shifts.append(last)
        raise Ic0Error(f"pivot breakdown at every shift in {[f'{s:.1e}' for s in shifts]}")
    nat.check(rc, "lg_ic0_factorize")
    l = CsrMatrix(n, l_rp, l_col[:nl], l_val[:nl])
    return Ic0Factor(l, shift.value, attempts.value)


class MulticolorIc0Factor:
    """FLAGGED, NON-REFERENCE preconditioner variant.

    IC(0) of P A P^T with P ordering the nodes by greedy colour
    (smallest-last) and then by id: every colour class is an independent
    set, so each triangular sweep has #colours dependency levels (C2 18,
    C3 78, C4 26 in the survey) instead of the natural order's 72 / 476 /
    227.  A different preconditioner than the reference's, hence different
    iteration counts (0.83-1.37x MVPs, survey-measured); the converged
    eigenpairs satisfy the same residual test.  Same .apply seam.
    """

    __slots__ = ("l", "shift", "attempts", "perm", "ncolors", "_dev")

    def __init__(self, l, shift, attempts, perm, ncolors):
        self.l = l
        self.shift = float(shift)
        self.attempts = int(attempts)
        self.perm = np.asarray(perm, dtype=np.int64)
        self.ncolors = int(ncolors)
        self._dev = None

    def device(self):
        if self._dev is None:
            self._dev = DeviceIc0(self.l, self.perm)
        return self._dev

    def apply(self, r):
        on_dev = dev.is_device_array(r)
        shape = tuple(r.shape) if on_dev else np.asarray(r).shape
        if shape != (self.l.n,):
            raise ValueError("vector length does not match factor dimension")
        z = self.device().apply(dev.to_device(r))
        return z if on_dev else dev.to_host(z)


def multicolor_order(a):
    """(perm, ncolors): nodes ordered by (smallest-last greedy colour, id)."""
    n = int(a.n)
    rp = np.ascontiguousarray(a.row_ptr, dtype=np.int64)
    ci = np.ascontiguousarray(a.col_idx, dtype=np.int64)
    color = np.empty(n, dtype=np.int32)
    nc = ctypes.c_int32()
    nat.call("lg_color_smallest_last", n, rp.ctypes.data, ci.ctypes.data if ci.size else None,
             color.ctypes.data, ctypes.byref(nc))
    perm = np.lexsort((np.arange(n), color)).astype(np.int64)
    return perm, nc.value


def permuted_matrix(a, perm):
    """P A P^T as a CsrMatrix (row i of the result is row perm[i] of a)."""
    n = int(a.n)
    inv = np.empty(n, dtype=np.int64)
    inv[perm] = np.arange(n)
    rows = inv[np.repeat(np.arange(n), np.diff(a.row_ptr))]
    cols = inv[a.col_idx]
    return CsrMatrix.from_coo(n, rows, cols, a.values, symmetric=True)


def ic0_factorize_multicolor(a, shift0=0.0, schedule=SHIFT_SCHEDULE):
    """FLAGGED variant: IC(0) of the multicolour-reordered matrix (same
    no-fill algorithm and shift ladder as ic0_factorize)."""
    perm, nc = multicolor_order(a)
    f = ic0_factorize(permuted_matrix(a, perm), shift0, schedule)
    return MulticolorIc0Factor(f.l, f.shift, f.attempts, perm, nc)


def identity_factor(n):
    """Factor whose application is the identity, for unpreconditioned runs."""
    return Ic0Factor(CsrMatrix.identity(n), 0.0, 0)


def precond_apply(f, r):
    """z = (L L^T)^{-1} r."""
    return f.apply(r)


def projected_precond_apply(f, q, r):
    """P M P r with P projecting out the columns held by q (ic0.py:144-150)."""
    return q.project_out(f.apply(q.project_out(r)))
