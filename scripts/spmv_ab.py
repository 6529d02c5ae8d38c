"""SpMV A/B on the benchmark graphs: device product vs the oracle's
restatement of the reference SpMV (sparse.py:128-139), and event time per
matvec with L2 flushed.  Development aid; run it once per library variant
(LG_LIB_OVERRIDE=path/to/variant.so).  Prints one JSON
line per graph."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200.generators import config_graph  # noqa: E402
from paper_1311_1695_b200.graphs import build_laplacian  # noqa: E402
from oracle import lapeig_oracle as O  # noqa: E402


def timed(step, reps=30, flush=True):
    junk = torch.empty(64 << 20, dtype=torch.float32, device="cuda")
    for _ in range(3):
        step()
    ts = []
    for _ in range(reps):
        if flush:
            junk.fill_(1.0)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        step()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


def main():
    names = sys.argv[1:] or ["C1", "C2", "C3", "C4", "C5"]
    mode = os.environ.get("LG_LIB_OVERRIDE", "default")
    for name in names:
        if name == "C5":
            from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
            A = rmat_laplacian_device(26, 16, seed=0)
            d = A.device()
            n = A.n
            x = dev.to_device(np.random.default_rng(0).standard_normal(n))
            y = dev.empty(n)
            ones = torch.ones(n, dtype=torch.float64, device="cuda")
            d.matvec(ones, y)
            torch.cuda.synchronize()
            rowsum = float(y.abs().max())      # L 1 = 0 exactly for integer weights
            us = timed(lambda: d.matvec(x, y), reps=10, flush=False)
            print(json.dumps({"graph": name, "mode": mode, "n": n, "nnz": A.nnz, "us": us,
                              "max_abs_L1": rowsum}), flush=True)
            del A, d, x, y, ones
            torch.cuda.empty_cache()
            continue
        g = config_graph(name)
        a = build_laplacian(g)
        d = a.device()
        xh = np.random.default_rng(0).standard_normal(a.n)
        x = dev.to_device(xh)
        y = dev.empty(a.n)
        d.matvec(x, y)
        torch.cuda.synchronize()
        yr = O.spmv(O.Csr(a.n, a.row_ptr, a.col_idx, a.values), xh)
        err = float(np.max(np.abs(y.cpu().numpy() - yr)) / np.max(np.abs(yr)))
        y2 = dev.empty(a.n)
        d.matvec(x, y2)
        torch.cuda.synchronize()
        det = bool(torch.equal(y, y2))
        us = timed(lambda: d.matvec(x, y))
        print(json.dumps({"graph": name, "mode": mode, "n": a.n, "nnz": a.nnz, "us": us,
                          "relerr": err, "deterministic": det}), flush=True)


if __name__ == "__main__":
    main()
