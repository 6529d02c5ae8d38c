"""Preconditioners on R-MAT graphs (dev aid): DACG / JD MVPs and wall time
with Jacobi (what C5 uses) vs FSAI, on host-generated R-MAT at a smaller
scale (the device C5 matrix has no host copy).  usage: scripts/rmat_prec.py 20"""
import json
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200.precond import JacobiFactor  # noqa: E402

scale = int(sys.argv[1]) if len(sys.argv) > 1 else 20
g, _ = L.largest_component(L.generators.rmat_graph(scale, 16, seed=0))
a = L.build_laplacian(g)
for name, mk in (("jacobi", lambda: JacobiFactor(a)), ("fsai32", lambda: L.fsai_factorize(a, 32))):
    t0 = time.perf_counter()
    f = mk()
    f.device()
    setup = time.perf_counter() - t0
    for sv, fn in (("dacg", L.dacg_smallest), ("jd", L.jd_smallest)):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        pairs, rep = fn(a, 5, delta=1e-8, f=f)
        torch.cuda.synchronize()
        print(json.dumps({"scale": scale, "n": a.n, "nnz": a.nnz, "prec": name, "solver": sv,
                          "setup_s": setup, "wall_s": time.perf_counter() - t0, "mvp": rep.mvp,
                          "eig": list(map(float, pairs.values))}), flush=True)
