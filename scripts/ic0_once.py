"""Warm up, then apply the C4 IC(0) factor once (ncu target; dev aid)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
a = L.build_laplacian(L.config_graph(name))
f = L.ic0_factorize_multicolor(a) if "--mc" in sys.argv else L.ic0_factorize(a)
d = f.device()
x = dev.to_device(np.random.default_rng(0).standard_normal(a.n)); z = dev.empty(a.n)
for _ in range(3): d.apply(x, z)
torch.cuda.synchronize()
torch.cuda.profiler.start()
d.apply(x, z)
torch.cuda.synchronize()
torch.cuda.profiler.stop()
print("ok")
