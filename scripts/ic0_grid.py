"""IC(0) apply time and parity vs the oracle for one grid size of the
dataflow sweep (LG_FLOW_GRID, dev aid).  usage: LG_FLOW_GRID=g python
scripts/ic0_grid.py C1 C2 ..."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402
from oracle import lapeig_oracle as O  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402

for name in sys.argv[1:]:
    a = L.build_laplacian(L.config_graph(name))
    f = L.ic0_factorize(a)
    d = f.device()
    xh = np.random.default_rng(0).standard_normal(a.n)
    x = dev.to_device(xh)
    z = dev.empty(a.n)
    for _ in range(3):
        d.apply(x, z)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(20):
        d.apply(x, z)
    e1.record()
    torch.cuda.synchronize()
    l = f.l
    zr = O.Ic0(a.n, l.row_ptr, l.col_idx, l.values).apply(xh)
    err = float(np.max(np.abs(z.cpu().numpy() - zr)) / np.max(np.abs(zr)))
    print(json.dumps({"graph": name, "grid": os.environ.get("LG_FLOW_GRID", "full"),
                      "levels": d.levels, "apply_us": e0.elapsed_time(e1) * 50,
                      "relerr": err}), flush=True)
