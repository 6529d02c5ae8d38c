"""Host-side profile of one DACG / JD solve after a warm-up solve (dev aid)."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import paper_1311_1695_b200 as L
name = sys.argv[1] if len(sys.argv) > 1 else "C4"
solver = sys.argv[2] if len(sys.argv) > 2 else "dacg"
a = L.build_laplacian(L.config_graph(name))
f = L.ic0_factorize_multicolor(a) if "--mc" in sys.argv else L.ic0_factorize(a)
fn = L.dacg_smallest if solver == "dacg" else L.jd_smallest
f.device()
fn(a, 5, delta=1e-8, f=f)
t0 = time.perf_counter()
pr = cProfile.Profile()
pr.enable()
pairs, rep = fn(a, 5, delta=1e-8, f=f)
pr.disable()
print("wall %.3f s" % (time.perf_counter() - t0), "report:", {k: v for k, v in vars(rep).items() if not hasattr(v, "__len__") or len(v) < 10})
pstats.Stats(pr).sort_stats(sys.argv[-1] if sys.argv[-1] in ("tottime", "cumulative") else "cumulative").print_stats(25)
