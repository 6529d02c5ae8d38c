"""IC(0) apply timing per config (dev aid)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    a = L.build_laplacian(L.config_graph(name))
    f = L.ic0_factorize(a)
    d = f.device()
    x = dev.to_device(np.random.default_rng(0).standard_normal(a.n))
    z = dev.empty(a.n)
    for _ in range(3): d.apply(x, z)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10): d.apply(x, z)
    e1.record(); torch.cuda.synchronize()
    from oracle import lapeig_oracle as O
    want = O.Ic0(a.n, f.l.row_ptr, f.l.col_idx, f.l.values).apply(x.cpu().numpy())
    err = np.max(np.abs(z.cpu().numpy() - want)) / np.max(np.abs(want))
    print(name, "levels", d.levels, "sweep depth", d.sweep_levels, "entries", d.sweep_entries,
          "(factor %d)" % (2 * (d.nnz_l - a.n)), "apply %.1f us" % (e0.elapsed_time(e1) * 100),
          "err vs oracle apply %.1e" % err, flush=True)
