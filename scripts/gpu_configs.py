"""BASELINE configs on the device vs golden reference results (dev aid)."""
import hashlib, json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L

def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays: h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()

for name in sys.argv[1:] or ["C1", "C2"]:
    ref = json.load(open(f"tests/golden/config_{name}.json"))
    t0 = time.time(); g = L.config_graph(name); tg = time.time() - t0
    t0 = time.time(); a = L.build_laplacian(g); tb = time.time() - t0
    t0 = time.time(); f = L.ic0_factorize(a); tf = time.time() - t0
    print(name, "n", a.n, "gen %.2fs build %.2fs factor %.2fs" % (tg, tb, tf),
          "csr==ref", sha(a.row_ptr, a.col_idx, a.values) == ref["csr_sha256"],
          "ic0==ref", sha(f.l.row_ptr, f.l.col_idx, f.l.values) == ref["ic0_sha256"], flush=True)
    for sv, rr in ref["solvers"].items():
        fn = {"dacg": L.dacg_smallest, "jd": L.jd_smallest, "irlm": L.irlm_smallest}[sv]
        torch.cuda.synchronize(); t0 = time.time()
        pairs, rep = fn(a, ref["neig"], delta=ref["delta"], f=f)
        torch.cuda.synchronize(); wall = time.time() - t0
        err = np.max(np.abs(pairs.values - rr["eigenvalues"]) / np.abs(rr["eigenvalues"]))
        th, rs = L.rayleigh_residuals(a, pairs.vectors)
        print("  %-5s mvp %5d (ref %5d)  eig relerr %.1e  maxres %.1e  wall %.3fs (ref %.2fs) x%.0f" % (
            sv, rep.mvp, rr["mvp"], err, rs.max(), wall, rr["wall_seconds"], rr["wall_seconds"] / wall), flush=True)
