"""Device-only graphs for BASELINE C5 (R-MAT scale 26, ~2e9 nonzeros).

C5 cannot be assembled by the reference and does not fit the
host-side numpy pipeline either, so sampling, canonicalisation, largest
component and the Laplacian all run on the device (csrc/lg_gen.cu,
lg_spmv.cu:lg_csr_laplacian_device).  The result is a DeviceLaplacian: it
quacks like a CsrMatrix for the device solvers and spmv (n, nnz, symmetric,
device(), diagonal()), but has no host arrays -- host-side IC(0) is not
available for it; use JacobiFactor or a device preconditioner.

The RNG is counter-based (splitmix64 of seed, edge, bit), so the graph is
reproducible but is not the same sample as generators.rmat_graph (numpy
default_rng); parity at this scale is residual-certified.
"""

import ctypes

import numpy as np

from . import _device as dev
from . import _native as nat
from .sparse import DeviceCsr


class DeviceLaplacian:
    """Unit-weight graph Laplacian held only on the device."""

    def __init__(self, n, m, handle, panels=True):
        self.n = int(n)
        self.m = int(m)
        self.symmetric = True
        self._dev = DeviceCsr.from_handle(handle, self.n, self.n + 2 * self.m)
        if panels:  # off when only row blocks of it are multiplied (N > 1)
            self._dev.auto_panels()

    @property
    def nnz(self):
        return self.n + 2 * self.m

    def device(self):
        return self._dev

    def diagonal(self):
        d = dev.empty(self.n)
        nat.call("lg_csr_diagonal", self._dev.handle, d.data_ptr())
        return dev.to_host(d)


def rmat_laplacian_device(scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=0, lcc=True,
                          panels=True):
    """Sample an R-MAT graph on the device, keep its largest component and
    assemble its Laplacian in the packed SpMV format.  panels=False skips the
    column panels of the full product (for row-partitioned use, where only
    row blocks of the operator are multiplied)."""
    dev.require_cuda()
    di, dj = ctypes.c_void_p(), ctypes.c_void_p()
    m = ctypes.c_int64()
    nat.call("lg_rmat_device", int(scale), int(edge_factor), float(a), float(b), float(c),
             ctypes.c_uint64(seed), ctypes.byref(di), ctypes.byref(dj), ctypes.byref(m))
    n = 1 << scale
    mm = m.value
    try:
        if lcc:
            nl, ml = ctypes.c_int64(), ctypes.c_int64()
            nat.call("lg_lcc_device", n, mm, ctypes.byref(di), ctypes.byref(dj),
                     ctypes.byref(nl), ctypes.byref(ml))
            n, mm = nl.value, ml.value
        h = ctypes.c_void_p()
        nat.call("lg_csr_laplacian_device", n, mm, di, dj, ctypes.byref(h))
    finally:
        nat.load().lg_free(di)
        nat.load().lg_free(dj)
    return DeviceLaplacian(n, mm, h, panels=panels)
