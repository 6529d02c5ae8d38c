"""GPU time of one DACG iteration graph vs host loop (dev aid)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200.dacg import _DacgPlan
from paper_1311_1695_b200._plan import Fused, Spmv
name = sys.argv[1] if len(sys.argv) > 1 else "C1"
a = L.build_laplacian(L.config_graph(name))
for lab, f in (("ic0", L.ic0_factorize(a)), ("mc", L.ic0_factorize_multicolor(a)), ("fsai", L.fsai_factorize(a, 32))):
    with dev.solver_stream() as st:
        pl = _DacgPlan(a, f, a.n, 11)
        pl.C[0] = 1.0 / np.sqrt(a.n)
        pl.k = 1
        x = dev.to_device(np.random.default_rng(0).standard_normal(a.n))
        pl.X[0].copy_(x / x.norm()); pl.X[1].copy_(pl.X[0])
        Spmv(pl.csr, pl.X[0], pl.AX[0])(); pl.AX[1].copy_(pl.AX[0])
        pl.G[0].copy_(pl.AX[0]); pl.G[1].copy_(pl.AX[0]); pl.P.zero_()
        pl.S.set(since=10, period=100, q=1.0, delta=-1.0)   # never a convergence halt
        g = pl.graph(0)
        for _ in range(3):
            pl.p_clear(); g()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(200):
            pl.p_clear(); g()
        e1.record(st); torch.cuda.synchronize()
        gpu = e0.elapsed_time(e1) / 200 * 1e3
        t0 = time.perf_counter()
        for _ in range(200):
            pl.p_clear(); g(); pl.S.fetch()
        host = (time.perf_counter() - t0) / 200 * 1e6
        # eager (no graph) for comparison
        L_ = pl.plan(0)
        t0 = time.perf_counter()
        for _ in range(200):
            pl.p_clear()
            for fn in L_: fn()
            pl.S.fetch()
        eager = (time.perf_counter() - t0) / 200 * 1e6
        # per-launch GPU time
        parts = []
        pl.p_clear()
        for i, fn in enumerate(L_):
            e0.record(st)
            for _ in range(50): fn()
            e1.record(st); torch.cuda.synchronize()
            parts.append(round(e0.elapsed_time(e1) / 50 * 1e3, 1))
        print(name, lab, "graph gpu %.1f us/iter, graph+fetch %.1f us, eager+fetch %.1f us" % (gpu, host, eager))
        print("   per launch (isolated, us):", [(type(fn).__name__, p) for fn, p in zip(L_, parts)])
