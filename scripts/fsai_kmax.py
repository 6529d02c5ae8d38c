import json, os, sys, time
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L
GOLD = {"C3": "C3n20", "C4": "C4n10"}
for cfg in ("C3", "C4"):
    gold = json.load(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden", f"config_{GOLD[cfg]}.json")))
    a = L.build_laplacian(L.config_graph(cfg))
    for k in (8, 16, 24, 32, 48):
        f = L.fsai_factorize(a, k); f.device()
        for sv, fn in (("dacg", L.dacg_smallest), ("jd", L.jd_smallest)):
            if sv not in gold["solvers"]: continue
            w = []
            for _ in range(2):
                torch.cuda.synchronize(); t0 = time.perf_counter()
                p, r = fn(a, gold["neig"], delta=gold["delta"], f=f)
                torch.cuda.synchronize(); w.append(time.perf_counter() - t0)
            print(cfg, k, sv, round(w[1], 3), r.mvp, f.g.nnz, flush=True)
