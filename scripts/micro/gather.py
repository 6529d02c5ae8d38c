"""Gather-only floor for the C4 column stream (dev aid): a torch index_select
of x by the packed columns is the simplest 'stream cols + gather x' kernel."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
a = L.build_laplacian(L.config_graph(sys.argv[1] if len(sys.argv) > 1 else "C4"))
col = torch.from_numpy(a.col_idx.astype(np.int64)).cuda()
col32 = col.to(torch.int32)
x = torch.randn(a.n, dtype=torch.float64, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
def t(fn, cold):
    for _ in range(3): fn()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(20)]; e1 = [torch.cuda.Event(enable_timing=True) for _ in range(20)]
    for i in range(20):
        if cold: flush.fill_(i)
        e0[i].record(); fn(); e1[i].record()
    torch.cuda.synchronize()
    return np.mean([p.elapsed_time(q) for p, q in zip(e0, e1)]) * 1e3
out = torch.empty(a.nnz, dtype=torch.float64, device="cuda")
print("index_select x[col] (gather + write nnz doubles): cold %.1f warm %.1f us" % (
    t(lambda: torch.index_select(x, 0, col, out=out), True), t(lambda: torch.index_select(x, 0, col, out=out), False)))
perm = torch.randperm(a.n, device="cuda")
colp = perm[col]
print("random relabel: cold %.1f warm %.1f us" % (
    t(lambda: torch.index_select(x, 0, colp, out=out), True), t(lambda: torch.index_select(x, 0, colp, out=out), False)))
srt = torch.sort(col).values
print("sorted cols (perfect locality): cold %.1f warm %.1f us" % (
    t(lambda: torch.index_select(x, 0, srt, out=out), True), t(lambda: torch.index_select(x, 0, srt, out=out), False)))
y = torch.empty(a.nnz, dtype=torch.float64, device="cuda")
print("pure copy nnz doubles: cold %.1f us" % t(lambda: y.copy_(out), True))
