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
    k = int(sys.argv[sys.argv.index("--k") + 1]) if "--k" in sys.argv else 1
    pl = _DacgPlan(a, f, a.n, 11)
    # deflation basis: the kernel vector plus k - 1 orthonormal columns
    # (a mid-solve iteration: k - 1 pairs already locked)
    Qm = np.linalg.qr(np.column_stack([np.ones(a.n)] + [np.random.default_rng(j).standard_normal(a.n)
                                                        for j in range(k - 1)]))[0]
    for j in range(k):
        pl.C[j] = torch.from_numpy(np.ascontiguousarray(Qm[:, j])).cuda()
    pl.k = k
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
