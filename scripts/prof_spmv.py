"""C4 SpMV / IC(0) launches for ncu (development aid)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200.generators import config_graph
from paper_1311_1695_b200.graphs import build_laplacian
from paper_1311_1695_b200.ic0 import ic0_factorize

name = sys.argv[1] if len(sys.argv) > 1 else "C4"
g = config_graph(name)
a = build_laplacian(g)
d = a.device()
x = dev.to_device(np.random.default_rng(0).standard_normal(a.n))
y = dev.empty(a.n)
for _ in range(5):
    d.matvec(x, y)
if "ic0" in sys.argv:
    f = ic0_factorize(a).device()
    for _ in range(3):
        f.apply(x, y)
torch.cuda.synchronize()
print("ok")
