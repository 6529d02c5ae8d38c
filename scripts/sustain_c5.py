import os, sys, time, subprocess, numpy as np, torch
sys.path.insert(0, "/root/repo")
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
A = rmat_laplacian_device(26, 16, seed=0)
d = A.device(); n = A.n
x = dev.to_device(np.random.default_rng(0).standard_normal(n)); y = dev.empty(n)
t_end = time.time() + 90
e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
while time.time() < t_end:
    e0.record()
    for _ in range(20): d.matvec(x, y)
    e1.record(); torch.cuda.synchronize()
    smi = subprocess.run(["nvidia-smi","--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active","--format=csv,noheader"],capture_output=True,text=True).stdout.strip()
    print(f"{e0.elapsed_time(e1)/20:.2f} ms/spmv  {smi}", flush=True)
