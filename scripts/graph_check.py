import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
a = L.build_laplacian(L.config_graph("C1"))
f = L.ic0_factorize_multicolor(a)
for rep in range(2):
    torch.cuda.synchronize(); t0 = time.perf_counter()
    pairs, r = L.dacg_smallest(a, 10, delta=1e-10, f=f)
    torch.cuda.synchronize(); print("dacg C1 mc", r.mvp, "%.3f s" % (time.perf_counter() - t0))
