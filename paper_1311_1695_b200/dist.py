"""Row-partitioned multi-GPU plumbing.

One process per GPU.  The Laplacian is split into contiguous row blocks of
(nearly) equal nonzeros; each rank owns its rows of A and its slice of
every n-vector.  A matvec needs the whole x, so each step exchanges the
slices in place (one batch of NCCL point-to-point transfers over NVSwitch;
gloo in the CPU tests) and multiplies the rank's row block, which keeps the
global column numbering; dot products are local partials reduced in rank
order (deterministic).
"""

import numpy as np


def partition_rows(row_ptr, nparts):
    """Split points (len nparts + 1) of contiguous row blocks with nearly
    equal nonzeros: binary search on row_ptr at r * nnz / P."""
    row_ptr = np.asarray(row_ptr)
    nnz = int(row_ptr[-1])
    cuts = [0]
    for r in range(1, nparts):
        cuts.append(int(np.searchsorted(row_ptr, r * nnz / nparts)))
    cuts.append(len(row_ptr) - 1)
    return cuts


class RowPartition:
    """Contiguous row blocks of nearly equal nonzeros (split points by binary
    search on the row pointers at r * nnz / P)."""

    def __init__(self, row_ptr, world):
        self.world = int(world)
        self.cuts = partition_rows(row_ptr, world)
        self.counts = [self.cuts[i + 1] - self.cuts[i] for i in range(world)]

    def rows(self, rank):
        return self.cuts[rank], self.cuts[rank + 1]


def local_operator(a, part, rank, flags=0):
    """Rank `rank`'s rows of the CsrMatrix-like `a` as an n x n device CSR
    whose other rows are absent from the schedule (global column numbers)."""
    from . import _native as nat
    from .sparse import DeviceCsr
    r0, r1 = part.rows(rank)
    lo, hi = int(a.row_ptr[r0]), int(a.row_ptr[r1])
    rp = np.zeros(a.n + 1, dtype=np.int64)
    rp[r0 + 1:r1 + 1] = np.asarray(a.row_ptr[r0 + 1:r1 + 1]) - lo
    rp[r1 + 1:] = hi - lo
    return DeviceCsr(a.n, rp, np.asarray(a.col_idx[lo:hi]), np.asarray(a.values[lo:hi]),
                     flags=flags | nat.LG_CSR_SKIP_EMPTY)


def device_row_ptr(dmat):
    """Stream row pointers (n + 1) of a device matrix (packed: off-diagonal)."""
    from . import _native as nat
    rp = np.empty(dmat.n + 1, dtype=np.int64)
    nat.call("lg_csr_row_ptr", dmat.handle, rp.ctypes.data)
    return rp


def local_operator_device(dmat, part, rank):
    """Like local_operator, cut on the device from a device-only packed
    matrix (C5 scale: no host copy of the graph exists)."""
    import ctypes

    from . import _native as nat
    from .sparse import DeviceCsr
    r0, r1 = part.rows(rank)
    h = ctypes.c_void_p()
    nat.call("lg_csr_row_block", dmat.handle, int(r0), int(r1), ctypes.byref(h))
    info = [ctypes.c_int64() for _ in range(4)] + [ctypes.c_int(), ctypes.c_int64()]
    nat.call("lg_csr_info", h, *[ctypes.byref(v) for v in info])
    return DeviceCsr.from_handle(h, dmat.n, info[1].value)


class SliceExchange:
    """Every rank sends its slice of x to every peer and receives theirs in
    place, as one batch of point-to-point transfers (one NCCL group over
    NVLink / NVSwitch; gloo in the CPU tests).  Slices may differ in length
    -- no padding, no packing, no copies; each rank moves exactly the
    (n - own) entries it lacks."""

    def __init__(self, dist, part, rank):
        self.dist = dist
        self.part = part
        self.rank = rank

    def __call__(self, x):
        d, part, me = self.dist, self.part, self.rank
        r0, r1 = part.rows(me)
        ops = []
        for p in range(part.world):
            if p == me:
                continue
            q0, q1 = part.rows(p)
            if r1 > r0:
                ops.append(d.P2POp(d.isend, x[r0:r1], p))
            if q1 > q0:
                ops.append(d.P2POp(d.irecv, x[q0:q1], p))
        if ops:
            for req in d.batch_isend_irecv(ops):
                req.wait()
        return x
