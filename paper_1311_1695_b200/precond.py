"""Device preconditioners behind the reference's preconditioner seam.

The reference accepts None, a callable, or any object with .apply(r)
(pcg.py:112-117, dacg.py:187).  The device solvers need an object with
apply_raw(r_ptr, z_ptr, skip, stream); device_preconditioner() adapts:

    Ic0Factor (this package or the reference's)  -> DeviceIc0 sweeps
    JacobiFactor (flagged, non-reference variant) -> diagonal scaling
    None                                          -> identity (a copy)
    any other object with .apply / callable       -> called on CUDA tensors
"""

import numpy as np

from . import _device as dev
from . import _native as nat
from ._plan import Fused

_cache = {}


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
    if isinstance(f, JacobiFactor):
        return f
    if hasattr(f, "l") and hasattr(f.l, "row_ptr"):
        hit = _cache.get(id(f))
        if hit is None or hit[0] is not f:
            hit = (f, DeviceIc0(f.l))
            _cache[id(f)] = hit
        return hit[1]
    fn = f if callable(f) else f.apply
    return CallablePrec(fn, n)
