"""Host-buffer SpMV on C4 (dev aid): public numpy spmv and the C-ABI
lg_spmv_host, median over 100 calls; run with LG_HOST_PIPE=0/1."""
import ctypes
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200 import _native as nat  # noqa: E402

a = L.build_laplacian(L.config_graph("C4"))
n = a.n
xh = np.random.default_rng(1).standard_normal(n)
yh = np.empty(n)
xd, yd = dev.empty(n), dev.empty(n)
args = (a.device().handle, xh.ctypes.data, yh.ctypes.data, ctypes.c_void_p(xd.data_ptr()),
        ctypes.c_void_p(yd.data_ptr()), ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))


def med(fn, reps=100):
    for _ in range(5):
        fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return np.median(ts) * 1e6, np.percentile(ts, 90) * 1e6


print("pipe", os.environ.get("LG_HOST_PIPE", "1"),
      "public us (med, p90) %.0f %.0f" % med(lambda: L.spmv(a, xh)),
      "cabi us %.0f %.0f" % med(lambda: nat.call("lg_spmv_host", *args)), flush=True)
