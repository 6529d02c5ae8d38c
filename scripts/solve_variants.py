"""Solver wall time / MVPs: reference IC(0) vs flagged variants (dev aid)."""
import sys, time, json, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
for name in sys.argv[1:] or ["C2", "C3", "C4"]:
    ref = json.load(open(f"tests/golden/config_{name}.json"))
    a = L.build_laplacian(L.config_graph(name))
    precs = {"ic0": L.ic0_factorize(a), "mc-ic0": L.ic0_factorize_multicolor(a), "jacobi": L.JacobiFactor(a)}
    for pn, f in precs.items():
        d = __import__("paper_1311_1695_b200.precond", fromlist=["x"]).device_preconditioner(f, a.n)
        x = dev.to_device(np.random.default_rng(0).standard_normal(a.n)); z = dev.empty(a.n)
        for _ in range(3): d.apply(x, z) if hasattr(d, "apply") else None
        torch.cuda.synchronize(); t0 = time.perf_counter()
        for _ in range(10): d.apply(x, z)
        torch.cuda.synchronize(); ta = (time.perf_counter() - t0) / 10
        for sv in ref["solvers"]:
            fn = {"dacg": L.dacg_smallest, "jd": L.jd_smallest, "irlm": L.irlm_smallest}[sv]
            torch.cuda.synchronize(); t0 = time.perf_counter()
            try:
                pairs, rep = fn(a, ref["neig"], delta=ref["delta"], f=f)
                torch.cuda.synchronize(); w = time.perf_counter() - t0
                err = np.max(np.abs(pairs.values - ref["solvers"][sv]["eigenvalues"]) / np.array(ref["solvers"][sv]["eigenvalues"]))
                print("%s %-6s %-4s apply %7.1f us  mvp %5d (ref %5d)  wall %.3fs (ref %.1fs)  err %.1e" % (
                    name, pn, sv, ta * 1e6, rep.mvp, ref["solvers"][sv]["mvp"], w, ref["solvers"][sv]["wall_seconds"], err), flush=True)
            except Exception as e:
                print(name, pn, sv, "ERR", repr(e)[:150], flush=True)
