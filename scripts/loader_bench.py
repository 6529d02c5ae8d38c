"""Graph file ingest speed (dev aid, CPU): the C4 edge list (4.96 M edges)
written as a text edge list and as Matrix Market, read by load_edge_list
(C++ parser) and -- when /root/reference is present -- by the reference's
Python parsers.  Prints one JSON line."""
import json
import os
import sys
import tempfile
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402

g = L.config_graph("C4")
d = tempfile.mkdtemp()
el = os.path.join(d, "c4.txt")
with open(el, "w") as fh:
    fh.write(f"{g.n_nodes}\n")
    fh.writelines(f"{i} {j} {w!r}\n" for i, j, w in zip(g.i.tolist(), g.j.tolist(),
                                                        g.w.tolist()))
out = {"edges": g.m, "bytes": os.path.getsize(el)}
t0 = time.perf_counter()
ours = L.load_edge_list(el)
out["ours_s"] = time.perf_counter() - t0
out["ours_ok"] = ours.pairs()[:3] == g.pairs()[:3] and ours.m == g.m
if os.path.isdir("/root/reference/pkg/src"):
    sys.path.insert(0, "/root/reference/pkg/src")
    from lapeig.graphs import load_edge_list as ref_load
    t0 = time.perf_counter()
    ref = ref_load(el)
    out["reference_s"] = time.perf_counter() - t0
    out["identical"] = bool((ref.i == ours.i).all() and (ref.j == ours.j).all()
                            and (ref.w == ours.w).all())
print(json.dumps(out))
