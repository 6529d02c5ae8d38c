"""Device solvers vs the golden reference results (development aid)."""
import json, sys, time
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import graphs

G = np.load("tests/golden/kat_graphs.npz")
R = json.load(open("tests/golden/kat_results.json"))["graphs"]
names = sys.argv[1:] or list(R)
for name in names:
    info = R[name]
    n = int(G[name + "_n"][0])
    g = graphs.EdgeList.from_canonical(n, G[name + "_i"], G[name + "_j"], G[name + "_w"])
    a = L.build_laplacian(g)
    f = L.ic0_factorize(a)
    out = [name]
    for sv, fn in (("dacg", L.dacg_smallest), ("jd", L.jd_smallest), ("irlm", L.irlm_smallest)):
        ref = info["solvers"][sv]
        t0 = time.time()
        try:
            pairs, rep = fn(a, info["neig"], delta=info["delta"], f=f)
            err = np.max(np.abs(pairs.values - ref["eigenvalues"]) / np.abs(ref["eigenvalues"]))
            out.append((sv, rep.mvp, ref["mvp"], "%.1e" % err, "%.2fs" % (time.time() - t0)))
        except Exception as e:
            import traceback; traceback.print_exc()
            out.append((sv, "ERR", repr(e)[:200]))
    print(*out, flush=True)
