"""SpMV with / without the fused epilogue (dots, Q^T y), graph-timed (dev aid)."""
import sys, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev
from paper_1311_1695_b200._plan import Graph, Slots, Spmv
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
a = L.build_laplacian(L.config_graph(name))
d = L.sparse.device_csr(a)
n = a.n
x, y, z = (torch.randn(n, dtype=torch.float64, device="cuda") for _ in range(3))
Q = torch.randn(8, n, dtype=torch.float64, device="cuda")
S = Slots(capacity=256)
S.add("r", 32)
res = S.s[S.idx["r"]:]
cases = {
    "plain": Spmv(d, x, y),
    "theta": Spmv(d, x, y, theta=0.5),
    "1 dot": Spmv(d, x, y, dots=[x], result=res),
    "2 dots": Spmv(d, x, y, dots=[x, z], result=res),
    "Q^T y k=5": Spmv(d, x, y, q=Q, nq=5, result=res),
}
for nm, f in cases.items():
    with dev.solver_stream() as st:
        g = Graph([f] * 20)
        for _ in range(3): g()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st); g(); e1.record(st); torch.cuda.synchronize()
        print(f"{name} {nm:10s} {e0.elapsed_time(e1) / 20 * 1e3:7.1f} us")
