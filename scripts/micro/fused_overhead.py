"""GPU cost of one small fused pass inside a CUDA graph (dev aid): 100
identical launches captured in one graph, per-launch time from events."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import Fused, Graph, Prog, Slots  # noqa: E402

with dev.solver_stream() as st:
    for n in (2000, 14729, 148531, 989777):
        S = Slots(capacity=256)
        S.add("d", 8)
        S.add("a")
        a, b, c = dev.to_device(np.ones(n)), dev.empty(n), dev.empty(n)
        p = Prog(S, skip=None)
        p.const("a", 1.0)
        p.build()
        cases = {
            "copy": lambda: Fused(n, outs=[dict(out=b, terms=[(a, 1.0)])]),
            "axpy+dot": lambda: Fused(n, outs=[dict(out=b, terms=[(a, 1.0), (c, 2.0)])],
                                      dots=[(1, None)], result=S.s[S.idx["d"]:]),
            "axpy+dot+prog": lambda: Fused(n, outs=[dict(out=b, terms=[(a, 1.0), (c, 2.0)])],
                                           dots=[(1, None)], result=S.s[S.idx["d"]:], prog=p),
        }
        for name, mk in cases.items():
            fs = [mk() for _ in range(100)]
            g = Graph(fs)
            for _ in range(3):
                g()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(10):
                g()
            e1.record(st)
            torch.cuda.synchronize()
            print(f"n={n:8d} {name:14s} {e0.elapsed_time(e1) / 1000 * 1e3:7.2f} us/launch "
                  f"(graph={'eager' if g.eager else 'captured'})", flush=True)
