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


def partition_rows(row_ptr, nparts, row_weight=0.0):
    """Split points (len nparts + 1) of contiguous row blocks with nearly
    equal cost: binary search on the cumulative cost at r * total / P, the
    cost of rows [0, i) being row_ptr[i] + row_weight * i (nonzeros, plus
    row_weight nonzero-equivalents per row for the per-row vector work of a
    solver iteration; 0: the SpMV alone, equal nonzeros)."""
    row_ptr = np.asarray(row_ptr)
    n = len(row_ptr) - 1
    cost = row_ptr.astype(np.float64)
    if row_weight:
        cost = cost + float(row_weight) * np.arange(n + 1, dtype=np.float64)
    total = float(cost[-1])
    cuts = [0]
    for r in range(1, nparts):
        cuts.append(int(np.searchsorted(cost, r * total / nparts)))
    cuts.append(n)
    return cuts


# Nonzero-equivalents of one row's vector work in a DACG / JD iteration on
# B200: the SpMV costs ~6 ps per nonzero (C5: 12.9 ms / 2.14e9), the fused
# passes ~113 ps per row (C5: 3.7 ms / 32.8 M rows), so a rank's iteration is
# balanced when nnz + 19 * rows is.  An nnz-balanced split leaves the ranks
# that own the many low-degree rows of a power-law graph with ~3x the vector
# work (C5 at 8 ranks: 11 M rows against 0.3 M).
SOLVER_ROW_WEIGHT = 19.0


class RowPartition:
    """Contiguous row blocks of nearly equal cost (split points by binary
    search on the row pointers; row_weight as in partition_rows)."""

    def __init__(self, row_ptr, world, row_weight=0.0):
        self.world = int(world)
        self.row_weight = float(row_weight)
        self.cuts = partition_rows(row_ptr, world, row_weight)
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


# ---------------------------------------------------------------------------
# Row-partitioned solvers: the execution context of one rank.
#
# Every solver vector stays n long on every rank, but each rank only computes
# its own row slice [r0, r1): fused vector passes run over the slice, their
# dot-product partials are summed over ranks (one all-reduce per pass, before
# the scalar program that reads them), the SpMV exchanges the slices of its
# input in place and multiplies the rank's row block (global column
# numbering), and the preconditioner is local (Jacobi, or block-Jacobi IC(0)
# of the rank's diagonal block: the natural-order IC(0) sweeps do not shard).
# Scalar programs run redundantly on every rank on identical inputs, so every
# rank takes the same branches and launches the same collectives.


class TorchBackend:
    """Collectives of one rank over torch.distributed (NCCL over NVLink /
    NVSwitch on the GPU box, gloo in CPU tests)."""

    def __init__(self, dist):
        self.dist = dist
        # NCCL collectives are stream-ordered and can be captured into the
        # solver's CUDA graphs; gloo's are host-synchronous
        try:
            self.graph_safe = dist.get_backend() == "nccl"
        except Exception:
            self.graph_safe = False

    def _host_staged(self, t):
        """gloo moves host memory only: CUDA tensors go through the host."""
        return not self.graph_safe and getattr(t, "is_cuda", False)

    def allreduce_(self, t, comm):
        if self._host_staged(t):
            h = t.cpu()
            self.dist.all_reduce(h)
            t.copy_(h)
            return
        self.dist.all_reduce(t)

    def exchange_(self, x, comm):
        if self._host_staged(x):
            h = x.cpu()
            SliceExchange(self.dist, comm.part, comm.rank)(h)
            x.copy_(h)
            return
        SliceExchange(self.dist, comm.part, comm.rank)(x)

    def exchange_start(self, x, comm):
        """Issue the slice exchange; returns the requests to wait on (NCCL
        runs it on its own stream, after the work already queued on the
        current stream)."""
        if self._host_staged(x):
            self.exchange_(x, comm)
            return []
        d, part, me = self.dist, comm.part, comm.rank
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
        return d.batch_isend_irecv(ops) if ops else []

    def exchange_wait(self, reqs, comm):
        for r in reqs:
            r.wait()

    def barrier(self, comm):
        self.dist.barrier()


class ThreadWorld:
    """Ranks simulated by threads of one process on one GPU (tests only):
    each rank runs on its own stream; all-reduce sums the ranks' tensors in
    rank order (deterministic, identical on every rank) and the exchange
    copies peer slices in place.  Kernels never wait on each other across
    ranks -- ranks meet only at host barriers."""

    def __init__(self, world):
        import threading
        self.world = int(world)
        self.bar = threading.Barrier(self.world)
        self.buf = [None] * self.world

    def _sync(self):
        import torch
        torch.cuda.current_stream().synchronize()

    def allreduce_(self, t, comm):
        self._sync()
        self.buf[comm.rank] = t
        self.bar.wait()
        acc = self.buf[0].clone()
        for p in range(1, self.world):
            acc += self.buf[p]
        self._sync()
        self.bar.wait()
        t.copy_(acc)

    def exchange_(self, x, comm):
        self._sync()
        self.buf[comm.rank] = x
        self.bar.wait()
        for p in range(self.world):
            if p != comm.rank:
                q0, q1 = comm.part.rows(p)
                x[q0:q1].copy_(self.buf[p][q0:q1])
        self._sync()
        self.bar.wait()

    def exchange_start(self, x, comm):
        self.exchange_(x, comm)
        return None

    def exchange_wait(self, reqs, comm):
        pass

    def barrier(self, comm):
        self._sync()
        self.bar.wait()


class RowComm:
    """One rank of a row-partitioned solve: its partition, rank and
    collective backend.  Pass it to dacg_smallest(..., comm=...).

        comm = RowComm.from_torch(a, torch.distributed)        # NCCL / gloo
    """

    def __init__(self, part, rank, backend, force_dist=False):
        self.part = part
        self.rank = int(rank)
        self.world = part.world
        self.r0, self.r1 = part.rows(self.rank)
        self.backend = backend
        # force_dist: run the row-partitioned code path even at one rank
        # (tests of the collectives' plumbing on a single GPU)
        self.force_dist = bool(force_dist)

    @property
    def graph_safe(self):
        """Collectives can be captured into CUDA graphs (NCCL)."""
        return bool(getattr(self.backend, "graph_safe", False))

    @classmethod
    def from_torch(cls, a, dist, row_weight=SOLVER_ROW_WEIGHT):
        """Rank of a row-partitioned solve over torch.distributed; the rows
        are split for a balanced solver iteration (SOLVER_ROW_WEIGHT)."""
        return cls(RowPartition(matrix_row_ptr(a), dist.get_world_size(), row_weight),
                   dist.get_rank(), TorchBackend(dist))

    @property
    def nl(self):
        return self.r1 - self.r0

    def allreduce_(self, t):
        if self.world > 1 or self.force_dist:
            self.backend.allreduce_(t, self)

    def exchange_(self, x):
        if self.world > 1:
            self.backend.exchange_(x, self)

    def barrier(self):
        if self.world > 1:
            self.backend.barrier(self)

    def exchange_start(self, x):
        return self.backend.exchange_start(x, self) if self.world > 1 else None

    def exchange_wait(self, reqs):
        if self.world > 1:
            self.backend.exchange_wait(reqs, self)

    def split_operator(self, a):
        """(inner, outer) halves of this rank's row block (lg_csr_split_cols):
        inner reads only the rank's own slice of x (and holds the diagonal),
        outer every other column; None when the block is not packed."""
        op = self.local_operator(a)
        if not op.packed:
            return None
        return split_cols(op, self.r0, self.r1)

    def solver_operator(self, a):
        """The operator a row-partitioned solver multiplies by: the split
        row block (interior product overlapped with the exchange) when it
        packs, else the plain row block."""
        from ._plan import SplitOp
        sp = self.split_operator(a)
        return SplitOp(*sp) if sp is not None else self.local_operator(a)

    def local_operator(self, a):
        """This rank's row block of `a` (host CsrMatrix or device-only)."""
        if hasattr(a, "row_ptr") and getattr(a, "col_idx", None) is not None:
            return local_operator(a, self.part, self.rank)
        return local_operator_device(a.device(), self.part, self.rank)

    def local_preconditioner(self, a, f):
        """The rank-local preconditioner for the solver seam `f`: None /
        'fsai' / an FsaiFactor -> FSAI as row-partitioned SpMVs (the same
        preconditioner at every N; device-built for device-only matrices);
        'block_ic0' -> block-Jacobi IC(0) of the diagonal block; 'jacobi' /
        a JacobiFactor -> its slice."""
        from .precond import FsaiFactor, Ic0JacobiFactor, JacobiFactor
        host = hasattr(a, "row_ptr") and getattr(a, "col_idx", None) is not None
        if f is None:
            f = "fsai"
        if isinstance(f, str):
            if f == "jacobi":
                f = JacobiFactor(a)
            elif f == "block_ic0" and not host:
                raise ValueError("block_ic0 needs the matrix on the host")
            elif f == "block_ic0":
                return BlockJacobiIc0(a, self)
            elif f == "fsai":
                # device-only matrices (one off-diagonal value) get the
                # device-built factor
                f = FsaiFactor(a) if host else FsaiFactor.from_device(a)
            else:
                raise ValueError(f"unknown distributed preconditioner {f!r}")
        if isinstance(f, JacobiFactor):
            return LocalJacobi(f, self.r0, self.r1)
        if isinstance(f, FsaiFactor):
            return DistFsai(f, self)
        if isinstance(f, Ic0JacobiFactor):
            return DistIc0Jacobi(f, self)
        if isinstance(f, (BlockJacobiIc0, DistFsai, DistIc0Jacobi)):
            return f
        raise ValueError("row-partitioned solves take an FsaiFactor, an Ic0JacobiFactor, a "
                         "JacobiFactor, 'fsai', 'jacobi' or 'block_ic0' as preconditioner (the "
                         "natural-order IC(0) sweeps do not shard, SURVEY 8(e))")


def split_cols(dmat, r0, r1):
    """Interior / exterior halves of a packed row-block operator."""
    import ctypes

    from . import _native as nat
    from .sparse import DeviceCsr
    hi, ho = ctypes.c_void_p(), ctypes.c_void_p()
    nat.call("lg_csr_split_cols", dmat.handle, int(r0), int(r1), ctypes.byref(hi),
             ctypes.byref(ho))
    out = []
    for h in (hi, ho):
        info = [ctypes.c_int64() for _ in range(4)] + [ctypes.c_int(), ctypes.c_int64()]
        nat.call("lg_csr_info", h, *[ctypes.byref(v) for v in info])
        out.append(DeviceCsr.from_handle(h, dmat.n, info[1].value))
    # the exterior half reads all of x but the rank's own slice: when x
    # exceeds L2 (C5) its product runs as column panels whose x slices stay
    # L2-resident, like the single-GPU product (accumulating, block rows only)
    out[1].auto_panels()
    return tuple(out)


def col_panel(dmat, c0, c1, with_diag):
    """Columns [c0, c1) of a packed operator, every row (lg_csr_col_panel)."""
    import ctypes

    from . import _native as nat
    from .sparse import DeviceCsr
    h = ctypes.c_void_p()
    nat.call("lg_csr_col_panel", dmat.handle, int(c0), int(c1), int(bool(with_diag)),
             ctypes.byref(h))
    info = [ctypes.c_int64() for _ in range(4)] + [ctypes.c_int(), ctypes.c_int64()]
    nat.call("lg_csr_info", h, *[ctypes.byref(v) for v in info])
    return DeviceCsr.from_handle(h, dmat.n, info[1].value)


def matrix_row_ptr(a):
    """Row pointers to balance on: host CSR arrays, or the device matrix's."""
    if hasattr(a, "row_ptr") and getattr(a, "col_idx", None) is not None:
        return np.asarray(a.row_ptr)
    return device_row_ptr(a.device())


class LocalJacobi:
    """A rank's slice of a JacobiFactor: z = r / diag on rows [r0, r1),
    applied to slice pointers."""

    def __init__(self, f, r0, r1):
        self.f = f
        self.n = r1 - r0
        self._dinv = f._dinv[r0:r1]

    def apply_raw(self, r, z, skip, stream):
        from . import _native as nat
        nat.check(nat.load().lg_diag_apply(self.n, self._dinv.data_ptr(), r, z, skip, stream),
                  "lg_diag_apply")


class BlockJacobiIc0:
    """Block-Jacobi IC(0) (flagged, non-reference): the
    reference's IC(0) (same shift ladder, bit-exact host factorization) of
    the rank's diagonal block A[r0:r1, r0:r1], applied by the device sweeps
    to the rank's slice -- no communication in the apply."""

    def __init__(self, a, comm):
        from .ic0 import ic0_factorize
        from .sparse import CsrMatrix
        r0, r1 = comm.r0, comm.r1
        rp = np.asarray(a.row_ptr)
        ci = np.asarray(a.col_idx)
        va = np.asarray(a.values)
        lo, hi = int(rp[r0]), int(rp[r1])
        rows = np.repeat(np.arange(r1 - r0), np.diff(rp[r0:r1 + 1]))
        keep = (ci[lo:hi] >= r0) & (ci[lo:hi] < r1)
        cols = ci[lo:hi][keep] - r0
        vals = va[lo:hi][keep]
        rr = rows[keep]
        brp = np.zeros(r1 - r0 + 1, dtype=np.int64)
        np.add.at(brp, rr + 1, 1)
        brp = np.cumsum(brp)
        self.block = CsrMatrix(r1 - r0, brp, cols, vals, symmetric=True)
        self.factor = ic0_factorize(self.block)
        self.n = r1 - r0
        self.shift = self.factor.shift
        self.attempts = self.factor.attempts

    def apply_raw(self, r, z, skip, stream):
        self.factor.device().apply_raw(r, z, skip, stream)


class DistIc0Jacobi:
    """The reference IC(0) factor applied by s Jacobi sweeps per triangle
    (precond.Ic0JacobiFactor) across ranks: every sweep is a row-partitioned
    product after the in-place slice exchange of its input, the D^{-1}
    scalings are rank-local -- the same preconditioner at every rank count,
    so the iteration counts do not depend on N (unlike block-Jacobi IC(0))."""

    def __init__(self, f, comm):
        from . import _device as dev
        self.f = f
        self.comm = comm
        self.s = f.sweeps
        self.dinv = local_operator(f.dinv, comm.part, comm.rank)
        self.bf = local_operator(f.bf, comm.part, comm.rank)
        self.bb = local_operator(f.bb, comm.part, comm.rank)
        self.t = [dev.zeros(f.n) for _ in range(3)]
        self.n = f.n

    def dist_steps(self, r, z, skip=None):
        from ._plan import Exchange, Spmv, SpmvAcc
        s = self.s
        t1, t2, p = self.t
        fw = [t1, t2]
        steps = [Spmv(self.dinv, r, fw[0], skip=skip)]
        for i in range(1, s + 1):
            steps += [Exchange(self.comm, fw[(i - 1) % 2]),
                      Spmv(self.dinv, r, fw[i % 2], skip=skip),
                      SpmvAcc(self.bf, fw[(i - 1) % 2], fw[i % 2], skip=skip)]
        y = fw[s % 2]

        def bw(i):
            return z if (s - i) % 2 == 0 else p

        steps.append(Spmv(self.dinv, y, bw(0), skip=skip))
        for i in range(1, s + 1):
            steps += [Exchange(self.comm, bw(i - 1)),
                      Spmv(self.dinv, y, bw(i), skip=skip),
                      SpmvAcc(self.bb, bw(i - 1), bw(i), skip=skip)]
        return steps


class DistFsai:
    """FSAI across ranks: z = G^T (G r) as two row-partitioned SpMVs, each
    after the in-place slice exchange of its input -- the same
    preconditioner at every rank count (no block-Jacobi loss), so the
    iteration counts do not depend on N."""

    def __init__(self, f, comm):
        from . import _device as dev
        self.f = f
        self.comm = comm
        if f.g is not None:
            self.g = local_operator(f.g, comm.part, comm.rank)
            self.gt = local_operator(f.gt, comm.part, comm.rank)
        else:   # built on the device (FsaiFactor.from_device): cut on the device
            f._ensure()
            self.g = local_operator_device(f._dg, comm.part, comm.rank)
            self.gt = local_operator_device(f._dgt, comm.part, comm.rank)
        self.t = dev.zeros(f.n)
        self.n = f.n

    def dist_steps(self, r, z, skip=None):
        from ._plan import Exchange, Spmv
        return [Exchange(self.comm, r), Spmv(self.g, r, self.t, skip=skip),
                Exchange(self.comm, self.t), Spmv(self.gt, self.t, z, skip=skip)]
