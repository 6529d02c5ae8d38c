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
