"""C5 per-rank SpMV at N ranks (dev aid): the rank's row block unsplit and
as interior + exterior halves, each timed alone on one GPU."""
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import SpmvAcc  # noqa: E402
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device  # noqa: E402
from paper_1311_1695_b200.dist import (RowPartition, device_row_ptr, local_operator_device,  # noqa: E402
                                       split_cols)

A = rmat_laplacian_device(26, 16, seed=0)
full = A.device()
n = A.n
x = dev.to_device(np.random.default_rng(0).standard_normal(n))
y = dev.empty(n)
rp = device_row_ptr(full)


def t(fn, reps=10):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for world in (2, 4, 8):
    part = RowPartition(rp, world)
    for r in sorted({0, world // 2, world - 1}):
        r0, r1 = part.rows(r)
        op = local_operator_device(full, part, r)
        inner, outer = split_cols(op, r0, r1)
        out = {"ranks": world, "rank": r, "rows": r1 - r0,
               "unsplit_ms": t(lambda: op.matvec(x, y)),
               "inner_ms": t(lambda: inner.matvec(x, y)),
               "outer_ms": t(lambda: SpmvAcc(outer, x, y)()),
               "inner_nnz": inner.nnz, "outer_nnz": outer.nnz}
        print(json.dumps(out), flush=True)
        del op, inner, outer
        torch.cuda.empty_cache()
