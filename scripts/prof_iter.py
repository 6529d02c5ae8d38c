"""One eager DACG iteration between cudaProfilerStart/Stop, for
`ncu --profile-from-start off` (dev aid)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200.dacg import _DacgPlan
from paper_1311_1695_b200._plan import Spmv
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
a = L.build_laplacian(L.config_graph(name))
f = L.ic0_factorize_multicolor(a) if "--mc" in sys.argv else L.ic0_factorize(a)
with dev.solver_stream() as st:
    pl = _DacgPlan(a, f, a.n, 11)
    pl.C[0] = 1.0 / np.sqrt(a.n)
    pl.k = 1
    x = dev.to_device(np.random.default_rng(0).standard_normal(a.n))
    pl.X[0].copy_(x / x.norm()); pl.X[1].copy_(pl.X[0])
    Spmv(pl.csr, pl.X[0], pl.AX[0])(); pl.AX[1].copy_(pl.AX[0])
    pl.G[0].copy_(pl.AX[0]); pl.G[1].copy_(pl.AX[0]); pl.P.zero_()
    pl.S.set(since=10, period=100, q=1.0, delta=-1.0)
    pl.p_clear()
    steps = pl.plan(0)
    for _ in range(3):
        pl.p_clear()
        for fn in steps: fn()
    torch.cuda.synchronize()
    pl.p_clear()
    torch.cuda.synchronize()
    torch.cuda.profiler.start()
    for fn in steps: fn()
    torch.cuda.synchronize()
    torch.cuda.profiler.stop()
print("ok", [type(fn).__name__ for fn in steps])
