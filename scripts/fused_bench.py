"""Bandwidth of lg_fused pass shapes (dev aid)."""
import sys, torch
sys.path.insert(0, ".")
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200._plan import Fused, Graph, Slots
for n in [int(x) for x in (sys.argv[1:] or ["1000000", "8000000"])]:
    a, b, c, o, o2 = (torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(5))
    Q = torch.randn(6, n, dtype=torch.float64, device="cuda")
    S = Slots(capacity=256)
    S.add("r", 32)
    S.add("cq", 8)
    res = S.s[S.idx["r"]:]
    cases = {
        "copy o=a": (Fused(n, outs=[dict(out=o, terms=[(a, 1.0)])]), 16),
        "dot a.b": (Fused(n, dots=[(a, b)], result=res), 16),
        "o=a+2b, o.o": (Fused(n, outs=[dict(out=o, terms=[(a, 1.0), (b, 2.0)])], dots=[(1, None)], result=res), 24),
        "o=a-Qc(k=5)": (Fused(n, outs=[dict(out=o, terms=[(a, 1.0)], upd=(Q, 5, S.p("cq")))]), 8 * 7),
        "Q^T a (k=5)": (Fused(n, blocks=[(Q, 5, a)], result=res), 8 * 6),
        "2 outs+3 dots": (Fused(n, outs=[dict(out=o, terms=[(a, 1.0), (b, 0.5)]), dict(out=o2, terms=[(c, 1.0), (b, -0.5)])],
                               dots=[(1, None), (2, None), (1, 2)], result=res), 40),
    }
    for name, (f, bpe) in cases.items():
      with dev.solver_stream() as st:
        g = Graph([f] * 20)   # device time only (host launch cost excluded)
        for _ in range(3): g()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        g()
        e1.record(st); torch.cuda.synchronize()
        us = e0.elapsed_time(e1) / 20 * 1e3
        print(f"n={n:>9} {name:16s} {us:8.1f} us  {bpe * n / us / 1e6:6.2f} TB/s")
