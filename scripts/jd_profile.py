import sys, os, time, cProfile, pstats
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_1311_1695_b200 as L
a = L.build_laplacian(L.config_graph("C4"))
f = L.fsai_factorize(a, 32); f.device()
L.jd_smallest(a, 10, delta=1e-8, f=f)
torch.cuda.synchronize()
pr = cProfile.Profile(); pr.enable()
t0 = time.perf_counter(); p, r = L.jd_smallest(a, 10, delta=1e-8, f=f); torch.cuda.synchronize()
pr.disable()
print("wall", time.perf_counter() - t0, "mvp", r.mvp, "outer", r.outer_its)
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
