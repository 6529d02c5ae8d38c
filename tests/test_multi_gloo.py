"""Host logic of the row-partitioned multi-GPU path, world_size 2 on gloo.

The device path (bench.py, N > 1) partitions rows by nonzeros, all-gathers x
every step and multiplies the local row block.  Here the same partition and
exchange run on CPU ranks with the oracle SpMV standing in for the kernel,
and the gathered result must equal the single-process product bit for bit.
"""

import os
import socket

import numpy as np
import pytest


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.dist import RowPartition, SliceExchange, partition_rows
    from paper_1311_1695_b200.generators import chung_lu_graph

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = chung_lu_graph(4000, 2.1, 5.0, max_degree=400, weighted=True, seed=5)
        rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
        n = g.n_nodes
        cuts = partition_rows(rp, world)
        r0, r1 = cuts[rank], cuts[rank + 1]
        counts = [cuts[i + 1] - cuts[i] for i in range(world)]
        x_full = np.random.default_rng(0).standard_normal(n)
        # each rank owns its slice of x; the step all-gathers it
        x = torch.zeros(n, dtype=torch.float64)
        x[r0:r1] = torch.from_numpy(x_full[r0:r1])
        part = RowPartition(rp, world)
        assert part.cuts == cuts and part.counts == counts
        SliceExchange(dist, part, rank)(x)
        xg = x.numpy()
        assert np.array_equal(xg, x_full)
        # local rows
        lo, hi = rp[r0], rp[r1]
        lrp = rp[r0:r1 + 1] - lo
        loc = O.Csr(r1 - r0, lrp, col[lo:hi], val[lo:hi])
        # oracle spmv needs a square operator: evaluate the row block directly
        y_loc = np.zeros(r1 - r0)
        nz = np.flatnonzero(np.diff(lrp) > 0)
        y_loc[nz] = np.add.reduceat(loc.val * xg[loc.col], lrp[nz])
        yt = torch.zeros(n, dtype=torch.float64)
        yt[r0:r1] = torch.from_numpy(y_loc)
        y = SliceExchange(dist, part, rank)(yt).numpy()
        want = O.spmv(O.Csr(n, rp, col, val), x_full)
        ok_y = np.array_equal(y, want)
        # balanced by nonzeros
        nnz_r = [int(rp[cuts[i + 1]] - rp[cuts[i]]) for i in range(world)]
        ok_bal = max(nnz_r) - min(nnz_r) <= 2 * int(np.diff(rp).max())   # each cut within a row
        # deterministic dot: local partials reduced in rank order
        part = torch.tensor([float(y_loc @ xg[r0:r1])], dtype=torch.float64)
        allp = [torch.zeros(1, dtype=torch.float64) for _ in range(world)]
        dist.all_gather(allp, part)
        dot = sum(float(p) for p in allp)
        ok_dot = abs(dot - float(want @ x_full)) <= 1e-10 * abs(float(want @ x_full))
        q.put((rank, ok_y, ok_bal, ok_dot))
    finally:
        dist.destroy_process_group()


def test_row_partitioned_spmv_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in procs)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_y, ok_bal, ok_dot in res:
        assert ok_y and ok_bal and ok_dot, (rank, ok_y, ok_bal, ok_dot)


def test_partition_rows_properties():
    from paper_1311_1695_b200.dist import partition_rows
    rp = np.array([0, 5, 5, 6, 20, 21, 30, 31, 40], dtype=np.int64)
    for p in (1, 2, 3, 4, 8):
        cuts = partition_rows(rp, p)
        assert cuts[0] == 0 and cuts[-1] == len(rp) - 1
        assert all(a <= b for a, b in zip(cuts, cuts[1:]))
        assert len(cuts) == p + 1


def test_row_partition_uneven_world3():
    """Three ranks with slices of different lengths (nnz-balanced cuts of a
    skewed graph): the in-place exchange still delivers every slice."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in procs)
    assert all(p.exitcode == 0 for p in procs)
    for rank, ok_y, ok_bal, ok_dot in res:
        assert ok_y and ok_bal and ok_dot, (rank, ok_y, ok_bal, ok_dot)


def _comm_worker(rank, world, port, q):
    """RowComm over gloo: the collectives a row-partitioned solver issues
    (slot all-reduce, in-place slice exchange) and the plan context's slice
    views, on CPU tensors."""
    import torch
    import torch.distributed as dist

    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.dist import RowComm
    from paper_1311_1695_b200.generators import chung_lu_graph
    from paper_1311_1695_b200.sparse import CsrMatrix

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = chung_lu_graph(3000, 2.1, 5.0, max_degree=300, seed=7)
        rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
        a = CsrMatrix(g.n_nodes, rp, col, val)
        comm = RowComm.from_torch(a, dist)
        n = a.n
        x_full = np.random.default_rng(1).standard_normal(n)
        # slot all-reduce of per-rank dot partials = the global dot
        part = torch.tensor([x_full[comm.r0:comm.r1] @ x_full[comm.r0:comm.r1], 1.0])
        comm.allreduce_(part)
        ok_red = (abs(float(part[0]) - x_full @ x_full) <= 1e-12 * (x_full @ x_full)
                  and float(part[1]) == world)
        # exchange completes a vector whose other slices hold garbage
        x = torch.full((n,), np.nan, dtype=torch.float64)
        x[comm.r0:comm.r1] = torch.from_numpy(x_full[comm.r0:comm.r1])
        comm.exchange_(x)
        ok_x = np.array_equal(x.numpy(), x_full)
        # the split (overlapped) form: issue, work on the own slice, wait
        x2 = torch.full((n,), np.nan, dtype=torch.float64)
        x2[comm.r0:comm.r1] = torch.from_numpy(x_full[comm.r0:comm.r1])
        reqs = comm.exchange_start(x2)
        own = float(x2[comm.r0:comm.r1].sum())          # interior work meanwhile
        comm.exchange_wait(reqs)
        ok_x = ok_x and np.array_equal(x2.numpy(), x_full) and np.isfinite(own)
        q.put((rank, ok_red, ok_x, comm.r0, comm.r1))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_row_comm_collectives_gloo(world):
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
    res = sorted(q.get(timeout=5) for _ in procs)
    assert all(p.exitcode == 0 for p in procs)
    assert [r[3] for r in res][0] == 0 and all(res[i][4] == res[i + 1][3] for i in range(world - 1))
    for rank, ok_red, ok_x, _, _ in res:
        assert ok_red and ok_x, (rank, ok_red, ok_x)


def test_block_jacobi_ic0_block_and_factor():
    """The block-Jacobi IC(0) of a rank is the reference IC(0) of the dense
    diagonal block A[r0:r1, r0:r1] (host factorization, no GPU needed)."""
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.dist import BlockJacobiIc0, RowComm, RowPartition
    from paper_1311_1695_b200.generators import chung_lu_graph
    from paper_1311_1695_b200.graphs import largest_component
    from paper_1311_1695_b200.sparse import CsrMatrix
    g, _ = largest_component(chung_lu_graph(800, 2.1, 5.0, max_degree=100, seed=3))
    rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    a = CsrMatrix(g.n_nodes, rp, col, val)
    dense = np.zeros((a.n, a.n))
    for r in range(a.n):
        dense[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
    part = RowPartition(rp, 3)
    for rank in range(3):
        comm = RowComm(part, rank, backend=None)
        bj = BlockJacobiIc0(a, comm)
        r0, r1 = comm.r0, comm.r1
        blk = np.zeros((r1 - r0, r1 - r0))
        b = bj.block
        for r in range(b.n):
            blk[r, b.col_idx[b.row_ptr[r]:b.row_ptr[r + 1]]] = b.values[b.row_ptr[r]:b.row_ptr[r + 1]]
        assert np.array_equal(blk, dense[r0:r1, r0:r1])
        lrp, lcol, lval, shift, att = O.ic0_factorize(O.Csr(b.n, b.row_ptr, b.col_idx, b.values),
                                                     use_c=False)
        assert np.array_equal(bj.factor.l.values.view(np.int64), lval.view(np.int64))


def test_partition_rows_cost_weighted():
    """row_weight > 0 balances nnz + row_weight * rows: on a power-law graph
    every block's cost is within one row of the mean, and the low-degree
    tail is no longer handed to one rank."""
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.dist import SOLVER_ROW_WEIGHT, partition_rows
    from paper_1311_1695_b200.generators import chung_lu_graph
    g = chung_lu_graph(20000, 2.1, 8.0, max_degree=3000, seed=2)
    rp, _, _ = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    for world in (2, 3, 8):
        cuts = partition_rows(rp, world, SOLVER_ROW_WEIGHT)
        cost = [int(rp[cuts[i + 1]] - rp[cuts[i]]) + SOLVER_ROW_WEIGHT * (cuts[i + 1] - cuts[i])
                for i in range(world)]
        maxrow = int(np.diff(rp).max()) + SOLVER_ROW_WEIGHT
        assert max(cost) - min(cost) <= 2 * maxrow
        assert cuts[0] == 0 and cuts[-1] == len(rp) - 1 and cuts == sorted(cuts)
    assert partition_rows(rp, 4) == partition_rows(rp, 4, 0.0)
