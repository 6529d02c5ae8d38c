"""Per-launch GPU time of one DACG iteration on a device-built R-MAT
Laplacian with the Jacobi preconditioner (dev aid: where a C5 iteration's
time goes).  usage: python scripts/dacg_iter_dev.py [scale=26] [k=6]"""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import Spmv  # noqa: E402
from paper_1311_1695_b200.dacg import _DacgPlan  # noqa: E402
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device  # noqa: E402
from paper_1311_1695_b200.precond import JacobiFactor  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
k = int(sys.argv[2]) if len(sys.argv) > 2 else 6
A = rmat_laplacian_device(scale, 16, seed=0)
f = JacobiFactor(A)
n = A.n
with dev.solver_stream() as st:
    pl = _DacgPlan(A, f, n, k + 1)
    rng = np.random.default_rng(0)
    for j in range(k):
        v = torch.as_tensor(rng.standard_normal(n), device="cuda")
        pl.C[j].copy_(v / v.norm())
    pl.k = k
    x = dev.to_device(rng.standard_normal(n))
    pl.X[0].copy_(x / x.norm())
    pl.X[1].copy_(pl.X[0])
    Spmv(pl.csr, pl.X[0], pl.AX[0])()
    pl.AX[1].copy_(pl.AX[0])
    pl.G[0].copy_(pl.AX[0])
    pl.G[1].copy_(pl.AX[0])
    pl.P.zero_()
    pl.S.set(since=10, period=100, q=1.0, delta=-1.0)
    g = pl.graph(0)
    for _ in range(3):
        pl.p_clear()
        g()
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        pl.p_clear()
        g()
    e1.record(st)
    torch.cuda.synchronize()
    print(f"scale {scale} n={n} k={k}: graph {e0.elapsed_time(e1) / 10:.2f} ms/iter", flush=True)
    L_ = pl.plan(0)
    pl.p_clear()
    for i, fn in enumerate(L_):
        e0.record(st)
        for _ in range(5):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        print(f"  launch {i:2d} {type(fn).__name__:10s} {e0.elapsed_time(e1) / 5:8.3f} ms", flush=True)
