"""Eigenvector parity on the large, clustered configurations (north star:
"subspace angles <= 1e-6 for clustered eigenvalues").

The reference's eigenvectors on C3 / C3n20 / C4 / C4n10 are too large to
commit, so tests/golden/make_vec_sketches.py (run in the build container,
importing the reference) stored a seeded Gaussian sketch S_ref = G^T U_ref
(G: n x 64) of every run.  Here the device solver runs with the reference's
settings and preconditioner (its IC(0) factor, bit-exact), and the principal
angles between span(G^T U_ref[:, c]) and span(G^T V[:, c]) -- which estimate
the angles between the full subspaces to within ~15 %
(tests/golden/sketch_C4n10_validation.json: reference DACG vs reference JD,
exact vs sketched) -- are held to 1e-6 for every cluster of eigenvalues
(consecutive relative gaps < 1e-2, e.g. C3n20's 0.351607 / 0.351616 /
0.351762) and for the whole k-dimensional subspace.  Eigenvalues are held to
1e-8 relative of the reference run's, residuals (recomputed by the CPU
oracle) to the solver tolerance.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

from oracle import lapeig_oracle as O

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
sys.path.insert(0, str(GOLDEN))
import make_vec_sketches as MS  # noqa: E402  (sketch constants and helpers)

pytestmark = [pytest.mark.gpu, pytest.mark.slow]

ANGLE_TOL = 1e-6
CLUSTER_GAP = 1e-2
RUNS = sorted(MS.RUNS)


@pytest.fixture(scope="module")
def problems():
    """Laplacian + reference IC(0) factor + sketch matrix per config (cached)."""
    import paper_1311_1695_b200 as L
    cache = {}

    def get(cfg):
        base = cfg[:2]
        if base not in cache:
            a = L.build_laplacian(L.config_graph(base))
            cache[base] = (L, a, L.ic0_factorize(a), MS.sketch_matrix(a.n))
        return cache[base]
    return get


@pytest.mark.parametrize("key", RUNS)
def test_cluster_subspace_angles(problems, key):
    cfg, solver = key.split(":")
    ref = np.load(GOLDEN / f"sketch_{cfg}_{solver}.npz")
    L, a, f, g = problems(cfg)
    assert a.n == int(ref["n"])
    neig, delta = int(ref["neig"]), float(ref["delta"])
    fn = L.dacg_smallest if solver == "dacg" else L.jd_smallest
    pairs, rep = fn(a, neig, delta=delta, f=f, seed=0)
    want = ref["values"]
    assert np.max(np.abs(pairs.values - want) / want) <= 1e-8
    _, rs = O.rayleigh_residuals(O.Csr(a.n, a.row_ptr, a.col_idx, a.values), pairs.vectors)
    assert np.all(rs <= delta * 1.0000001)
    s_ours = g.T @ np.asarray(pairs.vectors)
    s_ref = ref["sketch"]
    worst = 0.0
    for grp in MS.clusters(want, CLUSTER_GAP) + [list(range(neig))]:
        sine = MS.max_sine(s_ref[:, grp], s_ours[:, grp])
        worst = max(worst, sine)
        assert sine <= ANGLE_TOL, (key, grp, sine)
    print(f"{key}: mvp {rep.mvp} (reference {int(ref['mvp'])}), worst sketched sine {worst:.1e}")

