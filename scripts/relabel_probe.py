"""Does relabelling C4 (hubs first / BFS order) shorten the SpMV?  Times the
product on the original and relabelled Laplacians (dev probe)."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200.graphs import EdgeList  # noqa: E402

g = L.config_graph(sys.argv[1] if len(sys.argv) > 1 else "C4")
n = g.n_nodes
deg = np.bincount(g.i, minlength=n) + np.bincount(g.j, minlength=n)


def relabel(order):
    new = np.empty(n, dtype=np.int64)
    new[order] = np.arange(n)
    i, j = new[g.i], new[g.j]
    lo, hi = np.minimum(i, j), np.maximum(i, j)
    o = np.lexsort((hi, lo))
    return EdgeList(n, lo[o], hi[o], g.w[o])


def bfs_order():
    a = L.build_laplacian(g)
    rp, ci = a.row_ptr, a.col_idx
    seen = np.zeros(n, bool)
    out = []
    start = int(np.argmax(deg))
    seen[start] = True
    frontier = [start]
    while frontier:
        out.extend(frontier)
        nxt = []
        for v in frontier:
            nb = ci[rp[v]:rp[v + 1]]
            nb = nb[~seen[nb]]
            seen[nb] = True
            nxt.extend(nb.tolist())
        frontier = nxt
    return np.array(out + np.flatnonzero(~seen).tolist())


def t_spmv(gg):
    a = L.build_laplacian(gg)
    d = a.device()
    x = torch.randn(n, device="cuda", dtype=torch.float64)
    y = torch.empty_like(x)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    ts = []
    for it in range(30):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        d.matvec(x, y)
        e1.record()
        torch.cuda.synchronize()
        if it >= 5:
            ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


res = {"orig": t_spmv(g),
       "degree_desc": t_spmv(relabel(np.argsort(-deg, kind="stable"))),
       "bfs_from_hub": t_spmv(relabel(bfs_order()))}
perm = torch.as_tensor(np.random.default_rng(0).permutation(n), device="cuda")
x = torch.randn(n, device="cuda", dtype=torch.float64)
for _ in range(3):
    x.index_select(0, perm)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(20):
    x.index_select(0, perm)
e1.record()
torch.cuda.synchronize()
res["permute_pass_us"] = e0.elapsed_time(e1) / 20 * 1e3
print(json.dumps({k: round(v, 1) for k, v in res.items()}))
