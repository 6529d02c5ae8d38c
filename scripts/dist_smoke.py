"""Two processes on ONE GPU exercising bench.py's N > 1 code (dev aid):
launched by torchrun with gloo (host-side collectives; no kernel waits on
another rank), every rank on cuda:0.  Runs the row-partitioned SpMV step
(_OverlappedProduct) and solve_dist_block on C2 and prints rank 0's lines."""
import json
import os
import sys

import torch
import torch.distributed as dist

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200.dist import RowPartition, local_operator  # noqa: E402

torch.cuda.set_device(0)
dist.init_process_group("gloo")
rank, world = dist.get_rank(), dist.get_world_size()
a = L.build_laplacian(L.config_graph("C2"))
import numpy as np  # noqa: E402
part = RowPartition(a.row_ptr, world)
op = local_operator(a, part, rank)
prod = bench._OverlappedProduct(dist, part, rank, op)
xh = np.random.default_rng(0).standard_normal(a.n)
x = dev.to_device(xh)
r0, r1 = part.rows(rank)
x[:r0] = float("nan")
x[r1:] = float("nan")
y = dev.empty(a.n)
prod(x, y)
torch.cuda.synchronize()
want = L.spmv(a, xh)
err = float(np.max(np.abs(y[r0:r1].cpu().numpy() - want[r0:r1])))
sd = bench.solve_dist_block(a, dist=dist, world=world, rank=rank, neig=5, delta=1e-8)
if rank == 0:
    print(json.dumps({"spmv_max_err": err, "solve_dist": sd}))
dist.destroy_process_group()
