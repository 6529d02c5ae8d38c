"""Generate the golden fixtures from the reference implementation.

Runs ONLY in the build container (it imports the reference package from
/root/reference/pkg/src, read-only); the outputs are committed under
tests/golden/ so the GPU box never needs /root/reference.

    python tests/golden/make_golden.py [--big]

Fixtures (all from the reference's own code paths):
  kat_graphs.npz      edge lists of the reference's test fixture graphs
                      (path/cycle/complete/star/random/geometric generators)
  kat_results.json    per fixture graph: Laplacian CSR (small ones inline),
                      IC(0) factor summary, spmv / ic0-apply of seeded vectors,
                      DACG / JD / IRLM eigenvalues, MVP counts, iterations
  kat_arrays.npz      the arrays behind kat_results.json
  config_<C>.json     BASELINE configs: SHA-256 of the reference CSR arrays
                      and IC(0) factor, and solver results (eigenvalues,
                      MVPs) at the BASELINE settings
  config_<C>_vecs.npz eigenvectors of those runs (C1, C2)
"""

import argparse
import hashlib
import json
import platform
import sys
import time
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
sys.path.insert(0, str(REF))
sys.path.insert(1, str(ROOT))

import lapeig  # noqa: E402  (the reference, imported read-only)
from lapeig import generators as rgen  # noqa: E402
from lapeig.dacg import dacg_smallest  # noqa: E402
from lapeig.graphs import EdgeList, build_laplacian  # noqa: E402
from lapeig.ic0 import ic0_factorize  # noqa: E402
from lapeig.irlm import irlm_smallest  # noqa: E402
from lapeig.jd import jd_smallest  # noqa: E402
from lapeig.sparse import MvpCounter, spmv  # noqa: E402


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


def env():
    import scipy
    return {"numpy": np.__version__, "scipy": scipy.__version__,
            "python": platform.python_version(), "reference": lapeig.__version__}


KAT = {
    "P3": lambda: rgen.path_graph(3),
    "P4": lambda: rgen.path_graph(4),
    "P10w": lambda: rgen.path_graph(10, weight=2.5),
    "C4": lambda: rgen.cycle_graph(4),
    "C7": lambda: rgen.cycle_graph(7),
    "K3": lambda: rgen.complete_graph(3),
    "K6": lambda: rgen.complete_graph(6),
    "S4": lambda: rgen.star_graph(3),
    "S9": lambda: rgen.star_graph(8),
    "grid4x5": lambda: rgen.grid_graph(4, 5),
    "rand50": lambda: rgen.random_connected_graph(50, 60, seed=7),
    "rand200": lambda: rgen.random_connected_graph(200, 400, seed=3),
    "rand15": lambda: rgen.random_connected_graph(15, 10, seed=2),
    "geo1000": lambda: rgen.geometric_graph(1000, 0.05, seed=1),
}


def solver_runs(a, f, neig, delta, solvers=("dacg", "jd", "irlm"), seed=0):
    out = {}
    vecs = {}
    for name in solvers:
        c = MvpCounter()
        t0 = time.perf_counter()
        try:
            if name == "dacg":
                pairs, rep = dacg_smallest(a, neig, delta=delta, f=f, seed=seed, counter=c)
            elif name == "jd":
                pairs, rep = jd_smallest(a, neig, delta=delta, f=f, seed=seed, counter=c)
            else:
                pairs, rep = irlm_smallest(a, neig, delta=delta, f=f, seed=seed, counter=c)
        except Exception as exc:  # recorded, not fatal
            out[name] = {"error": f"{type(exc).__name__}: {exc}"}
            continue
        wall = time.perf_counter() - t0
        out[name] = {
            "eigenvalues": [float(v) for v in pairs.values],
            "residuals": [float(v) for v in pairs.residuals],
            "mvp": int(rep.mvp),
            "outer_its": int(rep.outer_its),
            "inner_its_total": int(rep.inner_its_total),
            "wall_seconds": wall,
            "config": {k: v for k, v in rep.config.items()
                       if isinstance(v, (int, float, str, list))},
        }
        vecs[name] = pairs.vectors
    return out, vecs


def make_kat():
    graphs, arrays, results = {}, {}, {}
    for name, fn in KAT.items():
        g = fn()
        graphs[f"{name}_n"] = np.array([g.n_nodes])
        graphs[f"{name}_i"] = g.i
        graphs[f"{name}_j"] = g.j
        graphs[f"{name}_w"] = g.w
        a = build_laplacian(g)
        f = ic0_factorize(a)
        rng = np.random.default_rng(123)
        x = rng.standard_normal(a.n)
        arrays[f"{name}_rp"] = a.row_ptr
        arrays[f"{name}_col"] = a.col_idx
        arrays[f"{name}_val"] = a.values
        arrays[f"{name}_lrp"] = f.l.row_ptr
        arrays[f"{name}_lcol"] = f.l.col_idx
        arrays[f"{name}_lval"] = f.l.values
        arrays[f"{name}_x"] = x
        arrays[f"{name}_spmv"] = spmv(a, x)
        arrays[f"{name}_ic0"] = f.apply(x)
        neig = min(3 if a.n < 8 else 5, a.n - 1)
        res, vecs = solver_runs(a, f, neig, 1e-8)
        for k, v in vecs.items():
            arrays[f"{name}_{k}_vecs"] = v
        results[name] = {"n": a.n, "nnz": a.nnz, "neig": neig, "delta": 1e-8,
                         "ic0_shift": f.shift, "ic0_attempts": f.attempts,
                         "csr_sha256": sha(a.row_ptr, a.col_idx, a.values),
                         "ic0_sha256": sha(f.l.row_ptr, f.l.col_idx, f.l.values),
                         "solvers": res}
        print(name, a.n, {k: v.get("mvp") for k, v in res.items()}, flush=True)
    np.savez_compressed(HERE / "kat_graphs.npz", **graphs)
    np.savez_compressed(HERE / "kat_arrays.npz", **arrays)
    (HERE / "kat_results.json").write_text(json.dumps({"env": env(), "graphs": results},
                                                      indent=1))


CONFIG_RUNS = {
    # BASELINE.json configs[0..3] solver settings
    "C1": dict(neig=10, delta=1e-10, solvers=("dacg", "jd", "irlm")),
    "C2": dict(neig=10, delta=1e-10, solvers=("dacg", "jd")),
    "C3": dict(neig=5, delta=1e-10, solvers=("jd",)),
    "C4": dict(neig=5, delta=1e-8, solvers=("jd", "dacg")),
    # the full BASELINE neig for C3 (20, JD) and C4 (10, DACG + JD)
    "C3n20": dict(neig=20, delta=1e-10, solvers=("jd",)),
    "C4n10": dict(neig=10, delta=1e-8, solvers=("dacg", "jd")),
}


def make_config(name):
    from paper_1311_1695_b200.generators import config_graph  # new generators
    g = config_graph(name[:2])
    # feed the reference the very same canonical edge list
    rg = EdgeList(g.n_nodes, g.i, g.j, g.w)
    t0 = time.perf_counter()
    a = build_laplacian(rg)
    tb = time.perf_counter() - t0
    t0 = time.perf_counter()
    f = ic0_factorize(a)
    tf = time.perf_counter() - t0
    x = np.random.default_rng(0).standard_normal(a.n)
    y = spmv(a, x)
    z = f.apply(x)
    spec = CONFIG_RUNS[name]
    res, vecs = solver_runs(a, f, spec["neig"], spec["delta"], spec["solvers"])
    out = {
        "env": env(), "config": name, "n": a.n, "m": g.m, "nnz": a.nnz,
        "edges_sha256": sha(g.i, g.j, g.w),
        "csr_sha256": sha(a.row_ptr, a.col_idx, a.values),
        "degree_sha256": sha(a.diagonal()),
        "ic0_sha256": sha(f.l.row_ptr, f.l.col_idx, f.l.values),
        "ic0_shift": f.shift, "ic0_attempts": f.attempts,
        "build_seconds": tb, "factor_seconds": tf,
        "spmv_x_seed0": {"sum": float(y.sum()), "norm": float(np.linalg.norm(y)),
                         "sha256": sha(y)},
        "ic0_apply_x_seed0": {"norm": float(np.linalg.norm(z)), "head": z[:8].tolist()},
        "neig": spec["neig"], "delta": spec["delta"], "solvers": res,
    }
    (HERE / f"config_{name}.json").write_text(json.dumps(out, indent=1))
    if name in ("C1", "C2"):
        np.savez_compressed(HERE / f"config_{name}_vecs.npz", **vecs)
    print(name, {k: (v.get("mvp"), v.get("wall_seconds")) for k, v in res.items()}, flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="C1,C2")
    ap.add_argument("--no-kat", action="store_true")
    args = ap.parse_args()
    if not args.no_kat:
        make_kat()
    for c in [c for c in args.configs.split(",") if c]:
        make_config(c)


if __name__ == "__main__":
    main()
