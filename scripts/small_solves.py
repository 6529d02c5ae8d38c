"""Wall time of the C1 / C2 solves (golden settings, reference IC(0)) -- dev
aid for the small-graph latency work.  Prints one JSON line per run."""
import json
import sys
import time
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1311_1695_b200 as L  # noqa: E402

runs = {"C1": ("dacg", "jd", "irlm"), "C2": ("dacg", "jd")}
fns = {"dacg": L.dacg_smallest, "jd": L.jd_smallest, "irlm": L.irlm_smallest}
for cfg in [c for c in sys.argv[1:]] or list(runs):
    gold = json.loads((ROOT / "tests" / "golden" / f"config_{cfg}.json").read_text())
    a = L.build_laplacian(L.config_graph(cfg))
    f = L.ic0_factorize(a)
    f.device()
    for name in runs[cfg]:
        walls = []
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pairs, rep = fns[name](a, gold["neig"], delta=gold["delta"], f=f)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        r = gold["solvers"][name]
        err = float(np.max(np.abs(pairs.values - r["eigenvalues"]) / np.abs(r["eigenvalues"])))
        print(json.dumps({"cfg": cfg, "solver": name, "wall_s": round(walls[1], 4), "mvp": rep.mvp,
                          "ref_mvp": r["mvp"], "us_per_mvp": round(1e6 * walls[1] / rep.mvp, 1),
                          "eig_relerr": err}), flush=True)
