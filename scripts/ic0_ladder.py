"""Reference IC(0) on the C5 family: device-built R-MAT
(edge factor 16, a, b, c = .57, .19, .19, LCC, unit weights) at one scale,
its host CSR exported from the device (lg_csr_export_host), the host C++
factorization (lg_ic0_factorize, bit-exact with ic0.py:48-116) timed with its
peak host RSS, the factor uploaded into the dataflow sweeps (DAG levels,
apply time), and -- with --solve -- DACG to 5 pairs at delta 1e-8 with the
reference IC(0) next to device FSAI.  One scale per process (run it under
`timeout`); prints one JSON line.
usage: python scripts/ic0_ladder.py SCALE [--solve]"""
import ctypes
import json
import resource
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200 import _native as nat  # noqa: E402
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device  # noqa: E402


class HostCsr:
    """Duck-typed CsrMatrix over exported arrays (no re-validation of
    billions of entries; the device builder already guarantees the form)."""

    def __init__(self, n, rp, col, val):
        self.n, self.row_ptr, self.col_idx, self.values = n, rp, col, val
        self.nnz = int(rp[-1])
        self.symmetric = True

    def diagonal(self):
        out = np.empty(self.n)
        rows = np.repeat(np.arange(self.n), np.diff(self.row_ptr))
        m = self.col_idx == rows
        out[rows[m]] = self.values[m]
        return out


def rss_gb():
    return resource.getrusage(resource.RUSAGE_SELF).ru_maxrss / 2**20


scale = int(sys.argv[1])
out = {"scale": scale, "edge_factor": 16}
t0 = time.perf_counter()
A = rmat_laplacian_device(scale, 16, seed=0)
torch.cuda.synchronize()
out.update(n=A.n, nnz=A.nnz, build_s=round(time.perf_counter() - t0, 2))
t0 = time.perf_counter()
rp = np.empty(A.n + 1, dtype=np.int64)
col = np.empty(A.nnz, dtype=np.int64)
val = np.empty(A.nnz, dtype=np.float64)
nat.call("lg_csr_export_host", A.device().handle, rp.ctypes.data, col.ctypes.data,
         val.ctypes.data)
out.update(export_s=round(time.perf_counter() - t0, 2), rss_after_export_gb=round(rss_gb(), 1))
print(json.dumps(out), flush=True)
a = HostCsr(A.n, rp, col, val)
t0 = time.perf_counter()
f = L.ic0_factorize(a)
out.update(factor_s=round(time.perf_counter() - t0, 1), shift=f.shift, attempts=f.attempts,
           nnz_l=int(f.l.nnz), rss_after_factor_gb=round(rss_gb(), 1))
print(json.dumps(out), flush=True)
del col, val
t0 = time.perf_counter()
d = f.device()
torch.cuda.synchronize()
out.update(sweep_setup_s=round(time.perf_counter() - t0, 1), levels=int(d.levels))
x = dev.to_device(np.random.default_rng(0).standard_normal(A.n))
z = dev.empty(A.n)
for _ in range(2):
    d.apply(x, z)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    d.apply(x, z)
e1.record()
torch.cuda.synchronize()
out.update(apply_ms=round(e0.elapsed_time(e1) / 5, 2))
print(json.dumps(out), flush=True)
if "--solve" in sys.argv:
    res = {}
    for lab, prec in (("ic0 (reference)", f), ("fsai kmax 32, device setup (flagged)",
                                                 L.FsaiFactor.from_device(A, kmax=32))):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pairs, rep = L.dacg_smallest(A, 5, delta=1e-8, f=prec)
        torch.cuda.synchronize()
        res[lab] = {"wall_s": round(time.perf_counter() - t0, 2), "mvp": rep.mvp,
                    "eigenvalues": pairs.values.tolist()}
    out["dacg_5_pairs"] = res
    print(json.dumps(out), flush=True)
