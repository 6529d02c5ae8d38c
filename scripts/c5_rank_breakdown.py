"""Per-launch GPU time of rank 0's row-partitioned DACG iteration on C5 at N ranks, collectives as no-ops (dev aid)."""
import sys, os
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, "scripts"))
import numpy as np, torch
from scaling_projection import NullBackend
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200._plan import Seq
from paper_1311_1695_b200.dacg import _DacgPlan
from paper_1311_1695_b200.dist import RowComm, RowPartition, matrix_row_ptr
from paper_1311_1695_b200.precond import JacobiFactor
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
A = rmat_laplacian_device(26, 16, seed=0); f = JacobiFactor(A); n = A.n
world = int(sys.argv[1]) if len(sys.argv) > 1 else 8
part = RowPartition(matrix_row_ptr(A), world)
comm = RowComm(part, 0, NullBackend())
with dev.solver_stream() as st:
    pl = _DacgPlan(A, f, n, 7, comm)
    rng = np.random.default_rng(0)
    for j in range(6):
        v = torch.as_tensor(rng.standard_normal(n), device="cuda"); pl.C[j].copy_(v / v.norm())
    pl.k = 6
    x = dev.to_device(rng.standard_normal(n))
    for b in (pl.X[0], pl.X[1], pl.AX[0], pl.AX[1], pl.G[0], pl.G[1], pl.P): b.copy_(x / x.norm())
    pl.S.set(since=10, period=100, q=1.0, delta=-1.0)
    L_ = pl.plan(0)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    pl.p_clear()
    tot = 0
    for i, fn in enumerate(L_):
        for _ in range(2): fn()
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(5): fn()
        e1.record(st); torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 5
        tot += ms
        kinds = [type(s).__name__ for s in (fn.steps if isinstance(fn, Seq) else [fn])]
        print(f"{i:2d} {ms:8.3f} ms  {kinds}", flush=True)
    print("sum", round(tot, 3))
