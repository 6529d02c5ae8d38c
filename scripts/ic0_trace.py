"""Per-level timing of the IC(0) sweeps (dev aid)."""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev, _native as nat
for name in [x for x in sys.argv[1:] if not x.startswith("--")] or ["C3"]:
    a = L.build_laplacian(L.config_graph(name))
    f = L.ic0_factorize_multicolor(a) if "--mc" in sys.argv else L.ic0_factorize(a); d = f.device()
    lib = nat.load()
    tot = lib.lg_ic0_trace(d.handle, 1, None, 0)
    x = dev.to_device(np.random.default_rng(0).standard_normal(a.n)); z = dev.empty(a.n)
    for _ in range(3): d.apply(x, z)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (tot + 2))()
    lib.lg_ic0_trace(d.handle, 1, buf, tot + 2)
    raw = np.array(buf[:], dtype=np.float64)
    sch = (ctypes.c_int * (4 * tot))()
    nf = lib.lg_ic0_schedule(d.handle, 0, sch, 4 * tot)
    sf = np.array(sch[:4 * nf]).reshape(nf, 4)
    nb = lib.lg_ic0_schedule(d.handle, 1, sch, 4 * tot)
    sb = np.array(sch[:4 * nb]).reshape(nb, 4)
    for lab, t, sc, cnt in (("fwd", raw[:nf], sf, raw[nf]), ("bwd", raw[nf + 1:nf + 1 + nb], sb, raw[nf + 1 + nb])):
        dt = np.diff(t) / 1e3
        print(name, lab, "segments", len(t), "total %.1f us" % ((t[-1] - t[0]) / 1e3),
              "inline stages (4 applies)", int(cnt))
        for kind in (0, 1):
            m = sc[1:, 1] == kind
            if m.any():
                print("   %s: n=%d mean %.2f us  median %.2f  max %.2f" % (
                    "narrow" if kind else "wide", m.sum(), dt[m].mean(), np.median(dt[m]), dt[m].max()))
        order = np.argsort(-dt)[:8]
        print("   slowest:", [(int(i + 1), round(float(dt[i]), 1), int(sc[i + 1, 0]), int(sc[i + 1, 1])) for i in order])
        # tasks vs time
        tk = sc[1:, 0]
        for lo, hi in ((1, 16), (17, 100), (101, 1000), (1001, 10**9)):
            m = (tk >= lo) & (tk <= hi)
            if m.any(): print("   tasks %d-%d: n=%d mean %.2f us" % (lo, hi, m.sum(), dt[m].mean()))
