"""Per-node GPU cost of small launches inside a CUDA graph (dev aid)."""
import sys, time, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200._plan import Fused, Graph, Prog, Slots
for n in (2000, 1000000):
    with dev.solver_stream() as st:
        S = Slots(); S.add("d", 8); S.set(d=1.0)
        v = [torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(4)]
        f_copy = Fused(n, outs=[dict(out=v[0], terms=[(v[1], 1.0)])])
        f_dot = Fused(n, dots=[(v[1], v[2])], result=S.s[S.idx["d"]:])
        f_upd = Fused(n, outs=[dict(out=v[0], terms=[(v[1], 1.0, S.p("d")), (v[2], -1.0)])], dots=[(1, None)], result=S.s[S.idx["d"] + 1:])
        p = Prog(S); p.const("a", 1.0); p.add("b", "a", "a"); p.build()
        for lab, fns in (("copy", [f_copy]), ("dot", [f_dot]), ("upd+dot", [f_upd]), ("prog", [p])):
            g = Graph(fns * 20)
            for _ in range(3): g()
            torch.cuda.synchronize()
            e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(20): g()
            e1.record(st); torch.cuda.synchronize()
            print("n=%d %-8s %.2f us per node (graph)" % (n, lab, e0.elapsed_time(e1) / 400 * 1e3), flush=True)
