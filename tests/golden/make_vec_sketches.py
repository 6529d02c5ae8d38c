"""Record Gaussian sketches of the reference's eigenvectors on the large configs.

Runs ONLY in the build container (imports the reference from
/root/reference/pkg/src, read-only).  The full eigenvector blocks of C3/C4
(24-80 MB per run) are too large to commit, so for every run we store

    S = G^T U            (SKETCH_COLS x k),   G = sketch_matrix(n)

with G a fixed seeded Gaussian n x SKETCH_COLS matrix that the GPU tests
regenerate (tests/test_ref_vectors.py).  The principal angles between the
column spaces of G^T U_c and G^T V_c estimate those between U_c and V_c
(an oblivious subspace embedding: for a c-dimensional cluster the sketched
sines are within a small constant factor of the true ones).  The estimator
is validated here on the reference's own DACG vs JD vectors (C4n10), where
the exact angles are available, and the result is written next to the
sketches (`validation`).

    python tests/golden/make_vec_sketches.py C4n10:dacg     # one run
    python tests/golden/make_vec_sketches.py --all          # every run, parallel

Output: tests/golden/sketch_<config>_<solver>.npz with
  values (k,), residuals (k,), sketch (SKETCH_COLS, k), mvp, n,
  and the eigenvalues checked against config_<config>.json.
"""

import json
import os
import subprocess
import sys
import time
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
ROOT = HERE.parent.parent
SKETCH_COLS = 64
SKETCH_SEED = 1311_1695

RUNS = {
    "C3:jd": dict(neig=5, delta=1e-10),
    "C3n20:jd": dict(neig=20, delta=1e-10),
    "C4:jd": dict(neig=5, delta=1e-8),
    "C4:dacg": dict(neig=5, delta=1e-8),
    "C4n10:dacg": dict(neig=10, delta=1e-8),
    "C4n10:jd": dict(neig=10, delta=1e-8),
}


def sketch_matrix(n, cols=SKETCH_COLS, seed=SKETCH_SEED):
    """The fixed n x cols Gaussian sketch (shared with tests/test_ref_vectors.py)."""
    return np.random.default_rng(seed).standard_normal((n, cols))


def run_one(key):
    sys.path.insert(0, "/root/reference/pkg/src")
    sys.path.insert(1, str(ROOT))
    from lapeig.dacg import dacg_smallest
    from lapeig.graphs import EdgeList, build_laplacian
    from lapeig.ic0 import ic0_factorize
    from lapeig.jd import jd_smallest
    from lapeig.sparse import MvpCounter
    from paper_1311_1695_b200.generators import config_graph

    cfg, solver = key.split(":")
    spec = RUNS[key]
    g = config_graph(cfg[:2])
    a = build_laplacian(EdgeList(g.n_nodes, g.i, g.j, g.w))
    f = ic0_factorize(a)
    c = MvpCounter()
    t0 = time.perf_counter()
    fn = dacg_smallest if solver == "dacg" else jd_smallest
    pairs, rep = fn(a, spec["neig"], delta=spec["delta"], f=f, seed=0, counter=c)
    wall = time.perf_counter() - t0
    gold = json.loads((HERE / f"config_{cfg}.json").read_text())["solvers"][solver]
    # single-threaded BLAS here (the golden run used 8 threads): same pairs to roundoff
    gv = np.asarray(gold["eigenvalues"])
    assert np.max(np.abs(gv - pairs.values) / gv) <= 1e-10, "run differs from golden"
    print(key, "mvp", rep.mvp, "golden mvp", gold["mvp"], flush=True)
    u = np.asarray(pairs.vectors, dtype=np.float64)
    s = sketch_matrix(a.n).T @ u
    out = HERE / f"sketch_{cfg}_{solver}.npz"
    np.savez_compressed(out, values=pairs.values, residuals=pairs.residuals, sketch=s,
                        mvp=np.int64(rep.mvp), n=np.int64(a.n), neig=np.int64(spec["neig"]),
                        delta=np.float64(spec["delta"]), wall_seconds=np.float64(wall))
    # full vectors kept out of git, only for the estimator validation below
    np.save(f"/tmp/refvec_{cfg}_{solver}.npy", u)
    print(key, "mvp", rep.mvp, "wall", round(wall, 1), "->", out.name, flush=True)


def clusters(values, rel_gap):
    """Maximal runs of ascending eigenvalues whose consecutive relative gaps are < rel_gap."""
    groups, cur = [], [0]
    for i in range(1, len(values)):
        if (values[i] - values[i - 1]) / abs(values[i]) < rel_gap:
            cur.append(i)
        else:
            groups.append(cur)
            cur = [i]
    groups.append(cur)
    return groups


def max_sine(a, b):
    """Sine of the largest principal angle between the column spaces of a and b."""
    qa, _ = np.linalg.qr(a)
    qb, _ = np.linalg.qr(b)
    return float(np.linalg.norm(qb - qa @ (qa.T @ qb), 2))


def validate(cfg="C4n10"):
    u = np.load(f"/tmp/refvec_{cfg}_dacg.npy")
    v = np.load(f"/tmp/refvec_{cfg}_jd.npy")
    su = np.load(HERE / f"sketch_{cfg}_dacg.npz")["sketch"]
    sv = np.load(HERE / f"sketch_{cfg}_jd.npz")["sketch"]
    vals = np.load(HERE / f"sketch_{cfg}_dacg.npz")["values"]
    rows = []
    for grp in clusters(vals, 1e-2) + [list(range(len(vals)))]:
        exact = max_sine(u[:, grp], v[:, grp])
        est = max_sine(su[:, grp], sv[:, grp])
        rows.append({"columns": grp, "exact_sine": exact, "sketched_sine": est})
    (HERE / f"sketch_{cfg}_validation.json").write_text(json.dumps(rows, indent=1))
    for r in rows:
        print(r)


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--all":
        env = dict(os.environ, OPENBLAS_NUM_THREADS="1", OMP_NUM_THREADS="1")
        procs = [subprocess.Popen([sys.executable, __file__, k], env=env) for k in RUNS]
        rc = [p.wait() for p in procs]
        assert not any(rc), rc
        validate()
    elif len(sys.argv) > 1 and sys.argv[1] == "--validate":
        validate()
    else:
        run_one(sys.argv[1])


if __name__ == "__main__":
    main()
