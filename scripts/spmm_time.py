"""Time lg_spmm_rowmajor (k columns, row-major) against k separate SpMVs."""
import json
import sys

import torch

import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200 import _native as nat

cfg = sys.argv[1] if len(sys.argv) > 1 else "C4"
a = L.build_laplacian(L.config_graph(cfg))
d = a.device()
s = torch.cuda.current_stream().cuda_stream
for k in (2, 4, 8, 10, 16):
    X = torch.randn(a.n, k, device="cuda", dtype=torch.float64)
    Y = torch.empty_like(X)
    cols = X.t().contiguous()
    outs = torch.empty_like(cols)
    ws = dev.workspace().handle

    def mm():
        nat.call("lg_spmm_rowmajor", d.handle, X.data_ptr(), Y.data_ptr(), k, ws, s)

    def sep():
        for j in range(k):
            d.matvec(cols[j], outs[j])

    res = {}
    for name, f in (("spmm", mm), ("spmv_x_k", sep)):
        for _ in range(3):
            f()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(20):
            f()
        e1.record()
        torch.cuda.synchronize()
        res[name] = e0.elapsed_time(e1) / 20 * 1e3
    mm()
    sep()
    torch.cuda.synchronize()
    err = (Y.t() - outs).abs().max().item()
    print(json.dumps({"config": cfg, "n": a.n, "nnz": a.nnz, "k": k, "spmm_us": round(res["spmm"], 1),
                      "k_spmv_us": round(res["spmv_x_k"], 1),
                      "speedup": round(res["spmv_x_k"] / res["spmm"], 2), "max_abs_diff": err}))
