"""Time to solution with the reference IC(0) vs the flagged FSAI and
multicolour-IC(0) / Jacobi-sweep IC(0) variants on the BASELINE configs (dev aid; one JSON line
per run).  usage: python scripts/solve_fsai.py C2 C3 C4"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402

GOLD = {"C2": "C2", "C3": "C3n20", "C4": "C4n10"}
for cfg in sys.argv[1:] or ["C2", "C3", "C4"]:
    gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                       f"config_{GOLD[cfg]}.json")))
    a = L.build_laplacian(L.config_graph(cfg))
    t0 = time.perf_counter()
    precs = {"ic0": L.ic0_factorize(a)}
    setup = {"ic0": time.perf_counter() - t0}
    for k, lv in ((32, 1), (8, 2), (16, 2), (32, 2)):
        t0 = time.perf_counter()
        precs[f"fsai{k}_l{lv}"] = L.fsai_factorize(a, kmax=k, levels=lv)
        setup[f"fsai{k}_l{lv}"] = time.perf_counter() - t0
    f0 = precs["ic0"]
    for sw in (1, 2, 3):
        t0 = time.perf_counter()
        precs[f"ic0_jacobi{sw}"] = L.ic0_jacobi_sweeps(f0, sw)
        setup[f"ic0_jacobi{sw}"] = setup["ic0"] + time.perf_counter() - t0
    only = os.environ.get("PRECS")
    if only:
        precs = {k: v for k, v in precs.items() if k in only.split(",")}
    for p in precs.values():
        p.device()
    for sv, fn in (("dacg", L.dacg_smallest), ("jd", L.jd_smallest)):
        if sv not in gold["solvers"]:
            continue
        ref = np.asarray(gold["solvers"][sv]["eigenvalues"])
        for name, f in precs.items():
            walls = []
            for _ in range(2):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                pairs, rep = fn(a, gold["neig"], delta=gold["delta"], f=f)
                torch.cuda.synchronize()
                walls.append(time.perf_counter() - t0)
            print(json.dumps({"cfg": GOLD[cfg], "solver": sv, "prec": name, "wall_s": walls[1],
                              "mvp": rep.mvp, "ref_mvp": gold["solvers"][sv]["mvp"],
                              "setup_s": setup[name],
                              "eig_relerr": float(np.max(np.abs(pairs.values - ref) / ref))}),
                  flush=True)
