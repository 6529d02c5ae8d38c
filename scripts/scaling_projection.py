"""Projected strong scaling of the row-partitioned DACG iteration (dev aid;
NOT a multi-GPU measurement -- only one GPU is available).

Each rank's local work is MEASURED: the rank's DACG iteration (its row block
of the SpMV as interior + exterior halves, its preconditioner share, every
fused pass over its slice, the scalar programs) is built with the real
row-partitioned plan and timed alone on one GPU with the collectives
replaced by no-ops; the max over ranks is taken.  The collectives are
MODELLED: per iteration the slice exchanges (1 for the SpMV, +2 for FSAI, +2S for
S-sweep IC(0))
move (N-1)/N x 8n bytes into each rank at the measured 770 GB/s NVLink peer
rate plus 10 us, and every dot-product pass costs one 15 us all-reduce.
As with NCCL, the N > 1 iteration is captured into CUDA graphs (collectives
included; tests/test_gpu_dist.py::test_nccl_collectives_captured_in_solver_graphs).  usage: python scripts/scaling_projection.py C4|C5 [--jacobi] [--ic0j S] [--nnz-split]"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import AllReduce, Exchange, ExchangeStart, Prog, Seq  # noqa: E402
from paper_1311_1695_b200.dacg import _DacgPlan  # noqa: E402
from paper_1311_1695_b200.dist import RowComm, RowPartition, matrix_row_ptr  # noqa: E402
from paper_1311_1695_b200.precond import JacobiFactor  # noqa: E402


class NullBackend:
    graph_safe = True   # as NCCL: the iteration is captured into CUDA graphs

    def allreduce_(self, t, comm):
        pass

    def exchange_(self, x, comm):
        pass

    def exchange_start(self, x, comm):
        return None

    def exchange_wait(self, reqs, comm):
        pass

    def barrier(self, comm):
        pass


def count_progs(plan):
    """Stand-alone scalar-program launches of an iteration (at N > 1 they
    cannot fold into the pass that produced their dots: the dots are
    all-reduced first)."""
    c = 0
    for step in plan:
        for s in (step.steps if isinstance(step, Seq) else [step]):
            for u in (s.steps if isinstance(s, Seq) else [s]):
                c += isinstance(u, Prog)
    return c


def prog_launch_us(slots_owner):
    """Device time of one stand-alone scalar-program launch inside a CUDA
    graph (20 in a row, median of 5)."""
    from paper_1311_1695_b200._plan import Graph
    p = Prog(slots_owner)
    p.const("pp_a", 1.0)
    p.add("pp_b", "pp_a", "pp_a")
    with dev.solver_stream():
        g = Graph([p] * 20)
        for _ in range(3):
            g()
        torch.cuda.synchronize()
        ts = []
        for _ in range(5):
            t0 = time.perf_counter()
            g()
            torch.cuda.synchronize()
            ts.append((time.perf_counter() - t0) / 20 * 1e6)
    return float(np.median(ts))


def count_collectives(plan):
    ex = ar = 0
    for step in plan:
        steps = step.steps if isinstance(step, Seq) else [step]
        for s in steps:
            if isinstance(s, Seq):
                for u in s.steps:
                    ex += isinstance(u, (Exchange, ExchangeStart))
                    ar += isinstance(u, AllReduce)
            ex += isinstance(s, (Exchange, ExchangeStart))
            ar += isinstance(s, AllReduce)
    return ex, ar


def rank_iteration_us(a, f, comm, k=6, iters=20):
    n = a.n
    with dev.solver_stream() as st:
        pl = _DacgPlan(a, f, n, k + 1, comm)
        rng = np.random.default_rng(0)
        for j in range(k):
            v = torch.as_tensor(rng.standard_normal(n), device="cuda")
            pl.C[j].copy_(v / v.norm())
        pl.k = k
        x = dev.to_device(rng.standard_normal(n))
        for buf in (pl.X[0], pl.X[1], pl.AX[0], pl.AX[1], pl.G[0], pl.G[1], pl.P):
            buf.copy_(x / x.norm())
        pl.S.set(since=10, period=100, q=1.0, delta=-1.0)
        g = pl.graph(0)
        for _ in range(3):
            pl.p_clear()
            g()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(iters):
            pl.p_clear()
            g()
        torch.cuda.synchronize()
        us = (time.perf_counter() - t0) / iters * 1e6
        ex, ar = count_collectives(pl.plan(0))
        npg = count_progs(pl.plan(0))
        tprog = prog_launch_us(pl.S) if npg else 0.0
    return us, ex, ar, npg, tprog


def main():
    cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
    if cfg == "C5":
        from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
        a = rmat_laplacian_device(26, 16, seed=0)
        if "--jacobi" in sys.argv:
            f, prec = JacobiFactor(a), "jacobi"
        else:
            from paper_1311_1695_b200.precond import FsaiFactor
            f, prec = FsaiFactor.from_device(a, kmax=32), "fsai"
        worlds = (1, 2, 4, 8)
    else:
        a = L.build_laplacian(L.config_graph(cfg))
        if "--ic0j" in sys.argv:
            sw = int(sys.argv[sys.argv.index("--ic0j") + 1])
            f = L.ic0_jacobi_sweeps(L.ic0_factorize(a), sw)
            prec = f"ic0_jacobi{sw} (reference IC(0) factor)"
        else:
            f = L.fsai_factorize(a, 32)
            prec = "fsai"
        worlds = (1, 2, 4, 8)
    rp = matrix_row_ptr(a)
    n = a.n
    base = None
    from paper_1311_1695_b200.dist import SOLVER_ROW_WEIGHT
    rw = 0.0 if "--nnz-split" in sys.argv else SOLVER_ROW_WEIGHT
    for world in worlds:
        part = RowPartition(rp, world, rw)
        ranks = range(world) if (cfg != "C5" or world <= 2) else (0, world // 2, world - 1)
        worst, ex, ar, npg, tprog = 0.0, 0, 0, 0, 0.0
        for r in ranks:
            comm = RowComm(part, r, NullBackend())
            us, ex, ar, npg, tprog = rank_iteration_us(a, f, comm)
            worst = max(worst, us)
            torch.cuda.empty_cache()
        comm_us = 0.0
        if world > 1:
            comm_us = ex * ((world - 1) / world * 8 * n / 770e9 * 1e6 + 10.0) + ar * 15.0
        total = worst + comm_us
        base = base or total
        rec = {"config": cfg, "preconditioner": prec, "ranks": world, "row_weight": rw,
               "local_us_measured": worst, "exchanges": ex, "allreduces": ar,
               "comm_us_modelled": comm_us, "iteration_us_projected": total,
               "speedup_projected": base / total, "efficiency_projected": base / total / world}
        if "--device-collectives" in sys.argv:
            # DESIGN 7 "device-side reductions": the finishing CTA of every
            # dot pass writes its partials into each peer's mailbox over
            # NVLink and sums the N mailboxes in rank order (~3 us: one
            # NVLink hop + the fan-in), then runs the scalar program itself
            # -- the stand-alone program launches disappear; the slice
            # exchange is issued by the producing kernel as P2P stores
            # (same bytes, ~3 us instead of NCCL's ~10 us launch latency)
            dev_comm = 0.0
            local_dev = worst
            if world > 1:
                dev_comm = ex * ((world - 1) / world * 8 * n / 770e9 * 1e6 + 3.0) + ar * 3.0
                local_dev = worst - npg * tprog
            dtot = local_dev + dev_comm
            base_d = getattr(main, "_base_d", None) or dtot
            main._base_d = base_d
            rec.update(device_collectives={
                "prog_launches_removed": npg if world > 1 else 0, "prog_launch_us": tprog,
                "local_us": local_dev, "comm_us_modelled": dev_comm,
                "iteration_us_projected": dtot, "speedup_projected": base_d / dtot,
                "efficiency_projected": base_d / dtot / world})
        print(json.dumps(rec), flush=True)


if __name__ == "__main__":
    main()
