"""Per-level latency of the dataflow IC(0) sweep (dev aid).

For each direction prints the spread of level completion times T(L) =
max done over tasks at level L, the mean per-level step T(L) - T(L-1), and
where a task's time goes: start -> inputs ready (waiting / gathering) and
ready -> done (reduce, divide, store).
"""
import ctypes, sys, numpy as np, torch
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
from paper_1311_1695_b200 import _device as dev, _native as nat
for name in [x for x in sys.argv[1:] if not x.startswith("--")] or ["C3"]:
    if name.startswith("grid"):   # e.g. grid300: a hub-free 300 x 300 grid
        k = int(name[4:])
        a = L.build_laplacian(L.generators.grid_graph(k, k))
    else:
        a = L.build_laplacian(L.config_graph(name))
    f = L.ic0_factorize_multicolor(a) if "--mc" in sys.argv else L.ic0_factorize(a)
    d = f.device()
    lib = nat.load()
    tot = lib.lg_ic0_flow_trace(d.handle, 1, None, 0)
    x = dev.to_device(np.random.default_rng(0).standard_normal(a.n)); z = dev.empty(a.n)
    for _ in range(3): d.apply(x, z)
    torch.cuda.synchronize()
    buf = (ctypes.c_ulonglong * (4 * tot))()
    lib.lg_ic0_flow_trace(d.handle, 1, buf, 4 * tot)
    rec = np.array(buf[:], dtype=np.int64).reshape(tot, 4)
    lv = rec[:, 0]
    # split fwd / bwd: the level sequence restarts at 0
    cut = int(np.flatnonzero(np.diff(lv) < 0)[0]) + 1 if (np.diff(lv) < 0).any() else tot
    for lab, r in (("fwd", rec[:cut]), ("bwd", rec[cut:])):
        if not len(r): continue
        t0 = r[:, 1].min()
        lvl, st, rd, dn = r[:, 0], r[:, 1] - t0, r[:, 2] - t0, r[:, 3] - t0
        nl = lvl.max() + 1
        T = np.full(nl, -1.0)
        np.maximum.at(T, lvl, dn.astype(float))
        step = np.diff(T)
        print(f"{name} {lab}: tasks {len(r)} levels {nl} span {dn.max()/1e3:.1f} us; "
              f"level step mean {step.mean()/1e3:.2f} median {np.median(step)/1e3:.2f} us")
        # a task's wait: from max(start, T(L-1)) to ready; compute: ready -> done
        prev = np.where(lvl > 0, T[np.maximum(lvl - 1, 0)], 0.0)
        crit = (dn == T[lvl])   # the level's last task
        w = rd - np.maximum(st, prev)
        c = dn - rd
        print(f"   last-of-level tasks: ready-after-prev-level {np.median(w[crit])/1e3:.2f} us (median), "
              f"ready->done {np.median(c[crit])/1e3:.2f} us; start before prev done: "
              f"{(st[crit] < prev[crit]).mean()*100:.0f}%")
        print(f"   all tasks: ready->done median {np.median(c)/1e3:.2f} p90 {np.percentile(c,90)/1e3:.2f} us")
        big = np.argsort(-step)[:6]
        print("   slowest level steps (L, us):", [(int(i + 1), round(float(step[i]) / 1e3, 2)) for i in big])
        if "--gaps" in sys.argv:
            W = int(sys.argv[sys.argv.index("--gaps") + 1])
            gap = st[W:] - dn[:-W]   # start of a warp's next task - done of this one
            for l in range(min(nl, 8)):
                m = (lvl[:-W] == l)
                print(f"     L{l}: done-start med {np.median(dn[:-W][m]-st[:-W][m])/1e3:.2f} us, "
                      f"gap to warp's next task med {np.median(gap[m])/1e3:.2f} p90 {np.percentile(gap[m],90)/1e3:.2f} us")
        if "--levels" in sys.argv:
            for l in range(nl):
                m = lvl == l
                print(f"     L{l:3d} tasks {m.sum():6d} T {T[l]/1e3:8.2f} step {(T[l]-(T[l-1] if l else 0))/1e3:6.2f} "
                      f"first start {st[m].min()/1e3:8.2f} ready med {np.median(rd[m]-st[m])/1e3:.2f} "
                      f"done-ready med {np.median(dn[m]-rd[m])/1e3:.2f}")
