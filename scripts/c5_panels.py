"""Column-panel SpMV probe on C5 (R-MAT 26): x (n*8 B) exceeds L2, so each
gather of the one-pass product misses to DRAM about half the time
(profiles/r01_spmv_c5_ncu_summary.txt).  Split the operator into P column
panels (lg_csr_col_panel) whose x slice fits in L2 and time y = P_0 x,
y += P_k x (lg_spmv_acc) against the one-pass product; CUDA events on the
launching stream, 10 timed products after 3 warm-ups."""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import SpmvAcc  # noqa: E402
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device  # noqa: E402
from paper_1311_1695_b200.dist import col_panel  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 26
plist = [int(v) for v in sys.argv[2].split(",")] if len(sys.argv) > 2 else [2, 4, 8, 16]
A = rmat_laplacian_device(scale, 16, seed=0)
d = A.device()
auto_p = d.npanels
d.set_panels(0)  # the one-pass baseline (DeviceLaplacian auto-panels x > 96 MiB)
n = A.n
x = dev.to_device(np.random.default_rng(0).standard_normal(n))
want = dev.empty(n)
y = dev.empty(n)
s = torch.cuda.current_stream()


def timed(fn, reps=10, warm=3):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


out = {"auto_panels": auto_p, "workload": f"R-MAT scale {scale} ef 16 LCC device-built", "n": n, "nnz": A.nnz,
       "x_mb": n * 8 / 2**20}
out["one_pass_ms"] = timed(lambda: d.matvec(x, want))
scale_ref = want.abs().max().item()
res = []
for P in plist:
    t0 = time.perf_counter()
    cuts = [n * k // P for k in range(P + 1)]
    panels = [col_panel(d, cuts[k], cuts[k + 1], k == 0) for k in range(P)]
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    accs = [SpmvAcc(p, x, y) for p in panels[1:]]

    def run():
        panels[0].matvec(x, y)
        for a in accs:
            a()
    ms = timed(run)
    err = (y - want).abs().max().item() / scale_ref
    nnz = [p.nnz for p in panels]
    res.append({"panels": P, "ms": ms, "speedup": out["one_pass_ms"] / ms, "rel_err": err,
                "build_s": build_s, "panel_nnz": nnz})
    print(json.dumps(res[-1]), flush=True)
    del accs, panels
    torch.cuda.synchronize()
    torch.cuda.empty_cache()
out["panels"] = res
print(json.dumps(out))
