"""C5 SpMV launches for ncu (dev aid): R-MAT scale 26 device build, 5 products."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device  # noqa: E402

A = rmat_laplacian_device(int(sys.argv[1]) if len(sys.argv) > 1 else 26, 16, seed=0)
d = A.device()
x = dev.to_device(np.random.default_rng(0).standard_normal(A.n))
y = dev.empty(A.n)
for _ in range(5):
    d.matvec(x, y)
torch.cuda.synchronize()
print("ok", A.n, A.nnz)
