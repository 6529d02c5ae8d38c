"""Probe: which cuSPARSE paths torch exposes here (fp64 CSR SpMV, CSR
triangular solve), timed on C4 next to lg_spmv / the IC(0) sweeps."""
import sys, time, json
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
import numpy as np, torch
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev

def ev_time(fn, reps=20, flush=None):
    s=[torch.cuda.Event(enable_timing=True) for _ in range(reps)]; e=[torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for _ in range(3): fn()
    torch.cuda.synchronize()
    for i in range(reps):
        if flush is not None: flush.fill_(i & 0xff)
        s[i].record(); fn(); e[i].record()
    torch.cuda.synchronize()
    return float(np.median([a.elapsed_time(b) for a,b in zip(s,e)]))*1e3

a = L.build_laplacian(L.config_graph("C4"))
flush = torch.empty(256<<20, dtype=torch.uint8, device="cuda")
x = torch.from_numpy(np.random.default_rng(0).standard_normal(a.n)).cuda()
out = {}
for idx in (torch.int32, torch.int64):
    try:
        A = torch.sparse_csr_tensor(torch.from_numpy(a.row_ptr).to(idx).cuda(), torch.from_numpy(a.col_idx).to(idx).cuda(),
                                    torch.from_numpy(a.values).cuda(), size=(a.n, a.n))
        y = A @ x
        yr = dev.to_host(L.spmv(a, x))
        out[f"spmv_{idx}"] = {"us": ev_time(lambda: A @ x, flush=flush), "maxdiff": float((y.cpu().numpy()-yr).__abs__().max())}
    except Exception as ex:
        out[f"spmv_{idx}"] = repr(ex)[:300]
d = a.device(); yy = dev.empty(a.n)
out["lg_spmv_us"] = ev_time(lambda: d.matvec(x, yy), flush=flush)
f = L.ic0_factorize(a)
Lt = torch.sparse_csr_tensor(torch.from_numpy(f.l.row_ptr).cuda(), torch.from_numpy(f.l.col_idx).cuda(), torch.from_numpy(f.l.values).cuda(), size=(a.n,a.n))
b = x.reshape(-1,1).contiguous()
for name, fn in [("triangular_solve", lambda: torch.triangular_solve(b, Lt, upper=False).solution),
                 ("linalg_solve_triangular", lambda: torch.linalg.solve_triangular(Lt, b, upper=False))]:
    try:
        z = fn(); torch.cuda.synchronize()
        out[name] = {"us": ev_time(fn, reps=10)}
    except Exception as ex:
        out[name] = repr(ex)[:300]
fd = f.device(); z = dev.empty(a.n)
out["lg_ic0_apply_us"] = ev_time(lambda: fd.apply(x, z), reps=10)
print(json.dumps(out, indent=1))
