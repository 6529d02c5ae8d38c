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
