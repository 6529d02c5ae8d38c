"""Row-partitioned DACG / JD on C4 (10 pairs, delta 1e-8, FSAI) with ranks
simulated by threads on one GPU (dist.ThreadWorld): the MVP counts and
eigenvalues at N = 1, 2, 4 (dev aid; timings of simulated ranks are not
meaningful and are not reported)."""
import json
import os
import sys
import threading

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200.dist import RowComm, RowPartition, ThreadWorld  # noqa: E402

a = L.build_laplacian(L.config_graph("C4"))
f = L.fsai_factorize(a, 32)
gold = json.load(open(os.path.join(os.path.dirname(__file__), "..", "tests", "golden",
                                   "config_C4n10.json")))["solvers"]
for name, fn in (("dacg", L.dacg_smallest), ("jd", L.jd_smallest)):
    ref = np.asarray(gold[name]["eigenvalues"])
    for world in (1, 2, 4):
        tw = ThreadWorld(world)
        part = RowPartition(a.row_ptr, world)
        out, errs = [None] * world, []

        def rank(r):
            try:
                torch.cuda.set_device(0)
                out[r] = fn(a, 10, delta=1e-8, f=f, comm=RowComm(part, r, tw))
            except BaseException as e:  # noqa: BLE001
                errs.append(e)
                tw.bar.abort()

        th = [threading.Thread(target=rank, args=(r,)) for r in range(world)]
        for t in th:
            t.start()
        for t in th:
            t.join()
        if errs:
            raise errs[0]
        pairs, rep = out[0]
        same = all(np.array_equal(o[0].values, pairs.values) for o in out)
        print(json.dumps({"solver": name, "ranks": world, "mvp": rep.mvp,
                          "ranks_agree": same,
                          "eig_relerr_vs_reference": float(np.max(np.abs(pairs.values - ref) / ref))}),
              flush=True)
