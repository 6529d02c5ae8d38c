"""IC(0) apply: dataflow sweeps vs the resident one-CTA sweep (dev aid).
Event time per apply, bitwise comparison of the two."""
import json, os, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev

def timed(d, x, z, reps=20):
    for _ in range(3): d.apply(x, z)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True); e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps): d.apply(x, z)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / reps

for name in sys.argv[1:] or ["C1", "C2", "C3"]:
    a = L.build_laplacian(L.config_graph(name))
    f = L.ic0_factorize(a)
    d = f.device()
    x = dev.to_device(np.random.default_rng(0).standard_normal(a.n))
    z0, z1 = dev.empty(a.n), dev.empty(a.n)
    auto = d.set_mode(-1)
    d.set_mode(0); t0 = timed(d, x, z0)
    d.set_mode(1); t1 = timed(d, x, z1)
    print(json.dumps({"graph": name, "n": a.n, "levels": d.levels, "auto_mode": auto,
                      "threads": os.environ.get("LG_SWEEP_CTA_THREADS", "512"),
                      "dataflow_us": round(t0, 1), "resident_us": round(t1, 1),
                      "same_bits": bool(torch.equal(z0, z1))}), flush=True)
