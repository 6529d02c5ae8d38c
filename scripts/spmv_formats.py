"""Plain vs packed SpMV timing + agreement (dev aid)."""
import sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200.sparse import DeviceCsr
from paper_1311_1695_b200 import _device as dev
for name in sys.argv[1:] or ["C1", "C2", "C3", "C4"]:
    a = L.build_laplacian(L.config_graph(name))
    x = dev.to_device(np.random.default_rng(0).standard_normal(a.n))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    res = {}
    for fl in (1, 0):
        d = DeviceCsr(a.n, a.row_ptr, a.col_idx, a.values, flags=fl)
        y = dev.empty(a.n)
        for _ in range(5): d.matvec(x, y)
        ts = []
        for cold in (True, False):
            e0 = [torch.cuda.Event(enable_timing=True) for _ in range(20)]
            e1 = [torch.cuda.Event(enable_timing=True) for _ in range(20)]
            for i in range(20):
                if cold: flush.fill_(i)
                e0[i].record(); d.matvec(x, y); e1[i].record()
            torch.cuda.synchronize()
            ts.append(np.mean([a_.elapsed_time(b_) for a_, b_ in zip(e0, e1)]) * 1e3)
        res[fl] = (y.clone(), ts, d.packed, d.stream_bytes)
        print(name, "packed" if d.packed else "plain ", "cold %.1f us warm %.1f us" % tuple(ts),
              "stream %.1f GB/s (cold)" % (d.stream_bytes / ts[0] / 1e3),
              "eff %.1f GB/s" % (d.algo_bytes / ts[0] / 1e3), flush=True)
    y0, y1 = res[1][0], res[0][0]
    print("  max rel diff", float((y0 - y1).abs().max() / y0.abs().max()))
