import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
a = L.build_laplacian(L.config_graph(sys.argv[1] if len(sys.argv) > 1 else "C4"))
f = L.ic0_factorize_multicolor(a); d = f.device()
x = dev.to_device(np.random.default_rng(0).standard_normal(a.n)); z = dev.empty(a.n)
for _ in range(3): d.apply(x, z)
torch.cuda.synchronize(); print("ok")
