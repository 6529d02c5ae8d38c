"""Fused vector passes at C5 size for ncu (dev aid): a 4-term linear
combination with 3 dots, and a block projection update v - Q c with k = 6
(the DACG deflation shape), n = 32.8 M."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import Fused, Slots  # noqa: E402

n = 32781264
k = 6
a, b, c, d = (dev.to_device(np.ones(n)) for _ in range(4))
out = dev.empty(n)
Q = torch.ones((k, n), dtype=torch.float64, device="cuda")
S = Slots(capacity=256)
S.add("r", 16)
S.add("cq", 8)
lin = Fused(n, outs=[dict(out=out, terms=[(a, 1.0), (b, 2.0), (c, 3.0), (d, 4.0)])],
            dots=[(1, None), (1, a), (a, b)], result=S.s[S.idx["r"]:])
proj = Fused(n, outs=[dict(out=out, terms=[(a, 1.0)], upd=(Q, k, S.p("cq")))],
             blocks=[(Q, k, 1)], result=S.s[S.idx["r"]:])
for _ in range(3):
    lin()
    proj()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for name, f, nbytes in (("lin4+3dots", lin, 5 * 8 * n), ("proj k=6 (+Q^T out)", proj, (2 + 2 * k) * 8 * n)):
    e0.record()
    for _ in range(10):
        f()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 100
    print(f"{name}: {us:.1f} us, {nbytes / us / 1e3:.0f} GB/s algorithmic", flush=True)
