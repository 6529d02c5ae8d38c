"""Device R-MAT + LCC + Laplacian (C5 pipeline) check (dev aid)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
from paper_1311_1695_b200 import _device as dev
for scale, ef in ((int(a.split(":")[0]), int(a.split(":")[1])) for a in (sys.argv[1:] or ["18:8"])):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    A = rmat_laplacian_device(scale, ef, seed=1)
    torch.cuda.synchronize(); tb = time.perf_counter() - t0
    d = A.device()
    x = dev.to_device(np.random.default_rng(0).standard_normal(A.n)); y = dev.empty(A.n)
    one = torch.ones(A.n, dtype=torch.float64, device="cuda")
    d.matvec(one, y); torch.cuda.synchronize()
    rowsum = float(y.abs().max())
    for _ in range(3): d.matvec(x, y)
    torch.cuda.synchronize()
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(10)]; e1 = [torch.cuda.Event(enable_timing=True) for _ in range(10)]
    for i in range(10):
        flush.fill_(i); e0[i].record(); d.matvec(x, y); e1[i].record()
    torch.cuda.synchronize()
    us = np.mean([p.elapsed_time(q) for p, q in zip(e0, e1)]) * 1e3
    # symmetry check: x^T (L y) == y^T (L x)
    z = dev.empty(A.n); d.matvec(y, z)
    w = dev.empty(A.n); d.matvec(x, w)
    s1 = float(torch.dot(x, z)); s2 = float(torch.dot(y, w))
    print("scale %d ef %d: n=%d m=%d nnz=%d build %.2fs  |L1|max=%.1e  sym %.1e  spmv %.1f us  stream %.0f GB/s eff %.0f GB/s" % (
        scale, ef, A.n, A.m, A.nnz, tb, rowsum, abs(s1 - s2) / abs(s1), us, d.stream_bytes / us / 1e3, d.algo_bytes / us / 1e3), flush=True)
