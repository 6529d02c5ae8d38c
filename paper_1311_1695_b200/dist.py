"""Row-partitioned multi-GPU plumbing.

One process per GPU.  The Laplacian is split into contiguous row blocks of
(nearly) equal nonzeros; each rank owns its rows of A and its slice of
every n-vector.  A matvec needs the whole x, so each step all-gathers the
slices (NCCL over NVLink on the B200 box, gloo in the CPU tests); dot
products are local partials reduced in rank order (deterministic).
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


class SliceGather:
    """All-gather of unequal row slices into a replicated vector.

    Collectives need equal-sized contributions, so each rank's slice is
    padded to the largest block, gathered into a (world, maxc) buffer and
    compacted back into x (a strided device copy).
    """

    def __init__(self, dist, counts, rank, like):
        import torch
        self.dist = dist
        self.counts = list(counts)
        self.rank = rank
        self.maxc = max(self.counts)
        self.offs = np.concatenate(([0], np.cumsum(self.counts))).tolist()
        self.send = torch.zeros(self.maxc, dtype=like.dtype, device=like.device)
        self.recv = torch.zeros(len(self.counts) * self.maxc, dtype=like.dtype,
                                device=like.device)

    def __call__(self, x):
        r = self.rank
        c = self.counts[r]
        self.send[:c].copy_(x[self.offs[r]:self.offs[r] + c])
        self.dist.all_gather_into_tensor(self.recv, self.send)
        blocks = self.recv.view(len(self.counts), self.maxc)
        for i, ci in enumerate(self.counts):
            if i != r:
                x[self.offs[i]:self.offs[i] + ci].copy_(blocks[i, :ci])
        return x


class RowPartition:
    """Row blocks of nearly equal nonzeros, with every n-vector kept in a
    padded layout: rank i's slice lives at [i*maxc, i*maxc + counts[i]) of
    a (world * maxc)-vector, so the SpMV's exchange is ONE in-place NCCL
    all-gather into the operand itself (no packing, no compaction copies)."""

    def __init__(self, row_ptr, world):
        self.world = int(world)
        self.cuts = partition_rows(row_ptr, world)
        self.counts = [self.cuts[i + 1] - self.cuts[i] for i in range(world)]
        self.maxc = max(self.counts) if self.counts else 0
        self.npad = self.world * self.maxc

    def padded_index(self, idx):
        idx = np.asarray(idx, dtype=np.int64)
        cuts = np.asarray(self.cuts, dtype=np.int64)
        owner = np.searchsorted(cuts, idx, side="right") - 1
        return owner * self.maxc + (idx - cuts[owner])

    def pad(self, v):
        """Host / device vector in natural order -> padded layout (zeros in the gaps)."""
        if hasattr(v, "new_zeros"):
            out = v.new_zeros(self.npad)
        else:
            out = np.zeros(self.npad, dtype=np.asarray(v).dtype)
        for i, c in enumerate(self.counts):
            out[i * self.maxc:i * self.maxc + c] = v[self.cuts[i]:self.cuts[i] + c]
        return out

    def unpad(self, vp):
        parts = [vp[i * self.maxc:i * self.maxc + c] for i, c in enumerate(self.counts)]
        if hasattr(vp, "new_zeros"):
            import torch
            return torch.cat(parts)
        return np.concatenate(parts)

    def local_rows(self, rank):
        """Padded index range of this rank's rows."""
        return rank * self.maxc, rank * self.maxc + self.counts[rank]


def local_operator(a, part, rank, flags=0):
    """Rank `rank`'s rows of the CsrMatrix-like `a` as an npad x npad device
    CSR in the padded index space (columns remapped, rows placed at the
    rank's padded slots, every other row absent from the schedule)."""
    from . import _native as nat
    from .sparse import DeviceCsr
    r0, r1 = part.cuts[rank], part.cuts[rank + 1]
    lo, hi = int(a.row_ptr[r0]), int(a.row_ptr[r1])
    p0 = rank * part.maxc
    rp = np.zeros(part.npad + 1, dtype=np.int64)
    rp[p0 + 1:p0 + (r1 - r0) + 1] = np.asarray(a.row_ptr[r0 + 1:r1 + 1]) - lo
    rp[p0 + (r1 - r0) + 1:] = hi - lo
    cols = part.padded_index(np.asarray(a.col_idx[lo:hi]))
    return DeviceCsr(part.npad, rp, cols, np.asarray(a.values[lo:hi]),
                     flags=flags | nat.LG_CSR_SKIP_EMPTY)


class PaddedAllGather:
    """In-place all-gather of the padded layout: each rank's slice is its
    contribution, the result lands in the same buffer."""

    def __init__(self, dist, part, rank):
        self.dist = dist
        self.part = part
        self.rank = rank

    def __call__(self, xpad):
        m = self.part.maxc
        self.dist.all_gather_into_tensor(xpad, xpad[self.rank * m:(self.rank + 1) * m])
        return xpad
