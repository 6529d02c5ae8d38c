"""Per-rank local SpMV time of the row-partitioned C5 operator, each rank's
block timed alone on this device (no exchange; dev aid for the N>1 path)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
from paper_1311_1695_b200.dist import RowPartition, device_row_ptr, local_operator_device
scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
A = rmat_laplacian_device(scale, 16, seed=0)
full = A.device()
rp = device_row_ptr(full)
xh = np.random.default_rng(0).standard_normal(A.n)
xp = dev.to_device(xh)
yp = dev.empty(A.n)
for world in (2, 4, 8):
    part = RowPartition(rp, world)
    ts = []
    for r in range(world):
        op = local_operator_device(full, part, r)
        for _ in range(2): op.matvec(xp, yp)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(5): op.matvec(xp, yp)
        e1.record(); torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) / 5)
        del op
        torch.cuda.empty_cache()
    print(f"world {world}: per-rank local SpMV ms {[round(t, 2) for t in ts]}  max {max(ts):.2f}  "
          f"x bytes received per rank <= {8 * (A.n - min(part.counts)) / 1e6:.0f} MB", flush=True)
