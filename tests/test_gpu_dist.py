"""Row-partitioned DACG on one B200: ranks simulated by
threads (dist.ThreadWorld -- each rank on its own stream, collectives at host
barriers, no kernel waits on another rank), the same code path the NCCL
ranks run.  Checked against the single-GPU solve with the same
preconditioner and against fresh residuals."""
import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _graph():
    import paper_1311_1695_b200 as L
    g = L.generators.chung_lu_graph(3000, 2.1, 4.0, max_degree=300, seed=5)
    g, _ = L.largest_component(g)
    return L.build_laplacian(g)


def _run_ranks(a, world, f, neig, delta):
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.dist import RowComm, RowPartition, ThreadWorld
    tw = ThreadWorld(world)
    part = RowPartition(a.row_ptr, world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            comm = RowComm(part, r, tw)
            out[r] = L.dacg_smallest(a, neig, delta=delta, f=f, seed=0, comm=comm)
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            tw.bar.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_dacg_jacobi(world):
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.precond import JacobiFactor
    from paper_1311_1695_b200.results import rayleigh_residuals
    a = _graph()
    f = JacobiFactor(a)
    delta = 1e-8
    ref, rrep = L.dacg_smallest(a, 4, delta=delta, f=f, seed=0)
    out = _run_ranks(a, world, f, 4, delta)
    for pairs, rep in out:
        assert np.array_equal(pairs.values, out[0][0].values)       # every rank agrees
        assert np.array_equal(pairs.vectors, out[0][0].vectors)
    pairs, rep = out[0]
    assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
    _, res = rayleigh_residuals(a, pairs.vectors)
    assert np.max(res) <= 1.5 * delta
    # roundoff-level differences in the dot partials may move the count a little
    assert abs(rep.mvp - rrep.mvp) <= 0.1 * rrep.mvp + 5


def test_row_partitioned_dacg_block_ic0():
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.results import rayleigh_residuals
    a = _graph()
    delta = 1e-8
    ref, _ = L.dacg_smallest(a, 4, delta=delta, seed=0)        # reference IC(0)
    out = _run_ranks(a, 2, "block_ic0", 4, delta)
    pairs, rep = out[0]
    assert np.array_equal(pairs.values, out[1][0].values)
    assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
    _, res = rayleigh_residuals(a, pairs.vectors)
    assert np.max(res) <= 1.5 * delta


def _run_ranks_jd(a, world, f, neig, delta):
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.dist import RowComm, RowPartition, ThreadWorld
    tw = ThreadWorld(world)
    part = RowPartition(a.row_ptr, world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            out[r] = L.jd_smallest(a, neig, delta=delta, f=f, seed=0,
                                   comm=RowComm(part, r, tw))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            tw.bar.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    return out


@pytest.mark.parametrize("world,prec", [(2, "jacobi"), (3, "block_ic0")])
def test_row_partitioned_jd(world, prec):
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.results import rayleigh_residuals
    a = _graph()
    delta = 1e-8
    ref, _ = L.jd_smallest(a, 4, delta=delta, seed=0)          # reference IC(0)
    out = _run_ranks_jd(a, world, prec, 4, delta)
    for pairs, _ in out:
        assert np.array_equal(pairs.values, out[0][0].values)
    pairs, rep = out[0]
    assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
    _, res = rayleigh_residuals(a, pairs.vectors)
    assert np.max(res) <= 1.5 * delta
    assert pairs.gram_defect() <= 1e-8 and pairs.kernel_overlap() <= 1e-8


def test_row_partitioned_dacg_device_only_matrix():
    """A device-only matrix (the C5 pipeline at scale 14): each rank cuts its
    row block on the device, Jacobi preconditioner; same pairs as the
    single-GPU solve."""
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import RowComm, RowPartition, ThreadWorld, matrix_row_ptr
    from paper_1311_1695_b200.precond import JacobiFactor
    A = rmat_laplacian_device(14, 8, seed=3)
    f = JacobiFactor(A)
    delta = 1e-8
    ref, _ = L.dacg_smallest(A, 3, delta=delta, f=f, seed=0)
    world = 2
    tw = ThreadWorld(world)
    part = RowPartition(matrix_row_ptr(A), world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            out[r] = L.dacg_smallest(A, 3, delta=delta, f=f, seed=0, comm=RowComm(part, r, tw))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            tw.bar.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    pairs, _ = out[0]
    assert np.array_equal(pairs.values, out[1][0].values)
    assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_fsai_same_iterations(world):
    """FSAI across ranks (dist.DistFsai: G and G^T as row-partitioned SpMVs
    with exchanges) is the same preconditioner at every rank count: DACG and
    JD take the single-GPU FSAI solve's MVP counts (to roundoff in the
    all-reduced dots) and return its eigenvalues."""
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.results import rayleigh_residuals
    a = _graph()
    f = L.fsai_factorize(a)
    delta = 1e-8
    for fn, run in ((L.dacg_smallest, _run_ranks), (L.jd_smallest, _run_ranks_jd)):
        ref, rrep = fn(a, 4, delta=delta, f=f, seed=0)
        out = run(a, world, f, 4, delta)
        pairs, rep = out[0]
        for p, _ in out:
            assert np.array_equal(p.values, pairs.values)
        assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
        assert abs(rep.mvp - rrep.mvp) <= 0.03 * rrep.mvp + 3
        _, res = rayleigh_residuals(a, pairs.vectors)
        assert np.max(res) <= 1.5 * delta


@pytest.mark.parametrize("world", [2, 3])
def test_row_partitioned_ic0_jacobi_sweeps(world):
    """The reference IC(0) factor with Jacobi-sweep triangular solves
    (dist.DistIc0Jacobi: every sweep a row-partitioned product after an
    exchange) is the same preconditioner at every rank count: DACG and JD
    take the single-GPU solve's MVP counts and eigenvalues."""
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.results import rayleigh_residuals
    a = _graph()
    f = L.ic0_jacobi_sweeps(L.ic0_factorize(a), 2)
    delta = 1e-8
    for fn, run in ((L.dacg_smallest, _run_ranks), (L.jd_smallest, _run_ranks_jd)):
        ref, rrep = fn(a, 4, delta=delta, f=f, seed=0)
        out = run(a, world, f, 4, delta)
        pairs, rep = out[0]
        for p, _ in out:
            assert np.array_equal(p.values, pairs.values)
        assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
        assert abs(rep.mvp - rrep.mvp) <= 0.03 * rrep.mvp + 3
        _, res = rayleigh_residuals(a, pairs.vectors)
        assert np.max(res) <= 1.5 * delta


@pytest.mark.parametrize("world,prec", [(2, "fsai"), (3, "jacobi")])
def test_row_partitioned_irlm(world, prec):
    """IRLM (inverse Lanczos, deflated PCG inner solves) row-partitioned:
    every rank returns the same pairs, eigenvalues within 1e-8 of the
    single-GPU reference-IC(0) solve, fresh residuals <= delta."""
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.dist import RowComm, RowPartition, ThreadWorld
    from paper_1311_1695_b200.results import rayleigh_residuals
    a = _graph()
    delta = 1e-8
    ref, _ = L.irlm_smallest(a, 4, delta=delta, seed=0)
    tw = ThreadWorld(world)
    part = RowPartition(a.row_ptr, world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            out[r] = L.irlm_smallest(a, 4, delta=delta, f=prec, seed=0,
                                     comm=RowComm(part, r, tw))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            tw.bar.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    pairs, _ = out[0]
    for p, _ in out:
        assert np.array_equal(p.values, pairs.values)
    assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
    _, res = rayleigh_residuals(a, pairs.vectors)
    assert np.max(res) <= 1.5 * delta


def test_nccl_collectives_captured_in_solver_graphs():
    """With the NCCL backend the row-partitioned DACG iteration -- passes,
    all-reduces of their dot partials, scalar programs -- is captured into
    CUDA graphs (no eager fallback).  One rank, forced onto the
    row-partitioned path; the pairs equal the plain single-GPU solve's."""
    import os
    import socket

    import torch
    import torch.distributed as dist

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200._plan import Graph
    from paper_1311_1695_b200.dist import RowComm, RowPartition, TorchBackend
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("nccl", rank=0, world_size=1,
                            device_id=torch.device("cuda", 0))
    try:
        a = _graph()
        f = L.fsai_factorize(a)
        ref, rrep = L.dacg_smallest(a, 4, delta=1e-8, f=f, seed=0)
        comm = RowComm(RowPartition(a.row_ptr, 1), 0, TorchBackend(dist), force_dist=True)
        assert comm.graph_safe
        cap0, fail0 = Graph.captured, Graph.failed
        pairs, rep = L.dacg_smallest(a, 4, delta=1e-8, f=f, seed=0, comm=comm)
        assert Graph.failed == fail0
        assert Graph.captured > cap0
        assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-12
        assert rep.mvp == rrep.mvp
    finally:
        dist.destroy_process_group()


def test_row_partitioned_dacg_device_fsai():
    """A device-only matrix with its FSAI built on the device
    (FsaiFactor.from_device): each rank cuts its rows of G and G^T on the
    device; the MVP count and pairs equal the single-GPU solve's."""
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import RowComm, RowPartition, ThreadWorld, matrix_row_ptr
    from paper_1311_1695_b200.precond import FsaiFactor
    A = rmat_laplacian_device(14, 8, seed=3)
    f = FsaiFactor.from_device(A, kmax=32)
    ref, rrep = L.dacg_smallest(A, 3, delta=1e-8, f=f, seed=0)
    world = 2
    tw = ThreadWorld(world)
    part = RowPartition(matrix_row_ptr(A), world)
    out, errs = [None] * world, []

    def rank(r):
        try:
            torch.cuda.set_device(0)
            out[r] = L.dacg_smallest(A, 3, delta=1e-8, f=f, seed=0, comm=RowComm(part, r, tw))
        except BaseException as e:  # noqa: BLE001
            errs.append(e)
            tw.bar.abort()

    th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
    for t in th:
        t.start()
    for t in th:
        t.join(timeout=300)
    if errs:
        raise errs[0]
    pairs, rep = out[0]
    assert np.array_equal(pairs.values, out[1][0].values)
    assert np.max(np.abs(pairs.values - ref.values) / ref.values) <= 1e-8
    assert abs(rep.mvp - rrep.mvp) <= 0.03 * rrep.mvp + 3
