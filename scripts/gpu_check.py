"""Quick device sanity check of the kernels against scipy (development aid)."""
import sys, time
import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla
import torch

from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200.generators import config_graph, path_graph
from paper_1311_1695_b200.graphs import build_laplacian
from paper_1311_1695_b200.ic0 import ic0_factorize
from paper_1311_1695_b200.sparse import spmv
from paper_1311_1695_b200._plan import Fused, Slots, Prog


def lap_ref(g):
    n = g.n_nodes
    deg = np.zeros(n)
    np.add.at(deg, g.i, g.w)
    np.add.at(deg, g.j, g.w)
    rows = np.concatenate([g.i, g.j, np.arange(n)])
    cols = np.concatenate([g.j, g.i, np.arange(n)])
    vals = np.concatenate([-g.w, -g.w, deg])
    o = np.lexsort((cols, rows))
    rp = np.zeros(n + 1, dtype=np.int64)
    np.add.at(rp, rows + 1, 1)
    return np.cumsum(rp), cols[o], vals[o]


for name in sys.argv[1:] or ["C1", "C4"]:
    g = config_graph(name) if name.startswith("C") else path_graph(5)
    t0 = time.time()
    a = build_laplacian(g)
    torch.cuda.synchronize()
    rp, ci, va = lap_ref(g)
    print(name, "n", a.n, "nnz", a.nnz, "build %.2fs" % (time.time() - t0),
          "bitexact", np.array_equal(rp, a.row_ptr), np.array_equal(ci, a.col_idx),
          np.array_equal(va.view(np.int64), a.values.view(np.int64)))
    S = sp.csr_matrix((a.values, a.col_idx, a.row_ptr), shape=(a.n, a.n))
    x = np.random.default_rng(0).standard_normal(a.n)
    y = spmv(a, x)
    yr = S @ x
    print("  spmv relerr", np.abs(y - yr).max() / np.abs(yr).max())
    d = a.device()
    print("  blocks", d.nblocks, "long", d.nlong)
    xd = dev.to_device(x); yd = dev.empty(a.n)
    for _ in range(3): d.matvec(xd, yd)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    reps = 50
    e0.record()
    for _ in range(reps): d.matvec(xd, yd)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    print("  spmv %.2f us  %.1f GB/s (algo bytes)" % (ms * 1e3, d.algo_bytes / ms / 1e6))
    # fused: dots and projection
    t = torch
    k = 3
    Q = t.randn(k, a.n, dtype=t.float64, device="cuda")
    S_ = Slots(); S_.add("c", 8); S_.add("d", 8)
    f1 = Fused(a.n, dots=[(xd, yd), (yd, None)], blocks=[(Q, k, yd)], result=S_.s[S_.idx["c"]:])
    f1()
    got = S_.s[:5].cpu().numpy()
    Qh = Q.cpu().numpy()
    want = np.concatenate([[x @ y, y @ y], Qh @ y])
    print("  fused dots relerr", np.abs(got - want).max() / np.abs(want).max())
    out = dev.empty(a.n)
    f2 = Fused(a.n, outs=[dict(out=out, terms=[(yd, 1.0), (xd, 2.0, S_.p("c"))], upd=(Q, k, S_.p("c", 2)))],
               dots=[(1, None)], result=S_.s[S_.idx["d"]:])
    f2()
    o = out.cpu().numpy()
    want2 = y + 2.0 * got[0] * x - Qh.T @ got[2:5]
    print("  fused update relerr", np.abs(o - want2).max() / np.abs(want2).max(),
          "norm2 relerr", abs(S_.s[S_.idx["d"]].item() - want2 @ want2) / (want2 @ want2))
    # IC0
    t0 = time.time()
    f = ic0_factorize(a)
    print("  ic0 factor %.2fs shift %g attempts %d" % (time.time() - t0, f.shift, f.attempts))
    L = sp.csr_matrix((f.l.values, f.l.col_idx, f.l.row_ptr), shape=(a.n, a.n))
    z = f.apply(x)
    yy = spla.spsolve_triangular(L, x, lower=True)
    zr = spla.spsolve_triangular(L.T.tocsr(), yy, lower=False)
    print("  ic0 apply relerr", np.abs(z - zr).max() / np.abs(zr).max(), "levels", f.device().levels)
    fd = f.device(); zd = dev.empty(a.n)
    for _ in range(3): fd.apply(xd, zd)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(20): fd.apply(xd, zd)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 20
    print("  ic0 apply %.2f us" % (ms * 1e3), "deterministic", torch.equal(zd, fd.apply(xd)))
    # scalar program
    p = Prog(S_)
    p.const("e", 3.0); p.const("f", 4.0); p.hypot("g", "e", "f"); p.sqrt("h", "g")
    p()
    print("  scalar", S_.read("g", "h"))
