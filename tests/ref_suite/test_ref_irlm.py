"""Restates the reference's pkg/tests/test_irlm.py against the drop-in:
ncv_for, LanczosState / inverse_lanczos_step / _thick_restart
(irlm.py:24-210) and the IRLM driver (irlm.py:230-292)."""

import numpy as np
import pytest

from lapeig.generators import (complete_graph, cycle_graph, path_graph, random_connected_graph,
                               star_graph)
from lapeig.graphs import build_laplacian
from lapeig.ic0 import ic0_factorize
from lapeig.irlm import LanczosState, _thick_restart, inverse_lanczos_step, irlm_smallest, ncv_for
from lapeig.pcg import kernel_basis
from lapeig.results import SolverError, rayleigh_residuals
from lapeig.sparse import MvpCounter
from tests.ref_suite.conftest import dense_positive_pairs

V2 = np.array([1.0, 0.0, -1.0]) / np.sqrt(2.0)


def setup(edges):
    a = build_laplacian(edges)
    return a, ic0_factorize(a), kernel_basis(a.n)


def centred_unit(n, seed):
    v = np.random.default_rng(seed).standard_normal(n)
    v -= v.mean()
    return v / np.linalg.norm(v)


# ---- ncv_for (test_irlm.py:30-53): host only ------------------------------
@pytest.mark.parametrize("neig,ncv", [(1, 15), (5, 30), (20, 60), (50, 120), (10, 40),
                                      (35, 90), (51, 122), (60, 140)])
def test_ncv_for_table(neig, ncv):
    """Anchors, interpolation and extrapolation (test_irlm.py:31-45)."""
    assert ncv_for(neig) == ncv


def test_ncv_for_monotone_and_positive():
    """test_irlm.py:47-53."""
    v = [ncv_for(k) for k in range(1, 81)]
    assert all(b >= a for a, b in zip(v, v[1:]))
    with pytest.raises(ValueError):
        ncv_for(0)


# ---- one Lanczos step (test_irlm.py:56-106) -------------------------------
@pytest.mark.gpu
def test_eigenvector_start_breaks_down():
    """The inverse maps v2 to itself: alpha = 1, breakdown, nothing
    pending, a further step raises (test_irlm.py:57-76)."""
    a, f, nb = setup(path_graph(3))
    st = LanczosState(V2, ncv=5)
    inverse_lanczos_step(st, a, f, 1e-12, nb)
    assert st.alpha[0] == pytest.approx(1.0, abs=1e-9)
    assert st.breakdown and not st.has_pending
    with pytest.raises(SolverError):
        inverse_lanczos_step(st, a, f, 1e-12, nb)


@pytest.mark.gpu
def test_generic_start_grows_and_interlaces():
    """test_irlm.py:78-93."""
    a, f, nb = setup(star_graph(4))
    st = LanczosState(centred_unit(a.n, 3), ncv=4)
    inverse_lanczos_step(st, a, f, 1e-12, nb)
    assert not st.breakdown and st.beta[0] > 0.0
    t1 = st.projected_matrix()[0, 0]
    inverse_lanczos_step(st, a, f, 1e-12, nb)
    mu = np.sort(np.linalg.eigvalsh(st.projected_matrix()))
    assert mu[0] <= t1 + 1e-12 <= mu[1] + 2e-12


@pytest.mark.gpu
def test_counter_charges_inner_iterations():
    """test_irlm.py:95-106."""
    a, f, nb = setup(random_connected_graph(12, extra_edges=8, seed=2))
    st = LanczosState(centred_unit(a.n, 0), ncv=6)
    c = MvpCounter()
    inverse_lanczos_step(st, a, f, 1e-8, nb, counter=c)
    assert c.count == st.last_inner_its > 0


# ---- the Lanczos relation (test_irlm.py:109-165) --------------------------
@pytest.mark.gpu
def test_projected_matrix_is_pinv_in_the_basis():
    """T_m = V' pinv(L) V, V orthonormal and kernel-free after 8 near-exact
    steps (test_irlm.py:110-145)."""
    a, f, nb = setup(random_connected_graph(25, extra_edges=15, seed=4))
    st = LanczosState(centred_unit(a.n, 7), ncv=10)
    for _ in range(8):
        inverse_lanczos_step(st, a, f, 1e-13, nb)
    cols = np.column_stack(st.columns)
    vm = cols[:, :st.m]
    assert np.max(np.abs(st.projected_matrix() - vm.T @ np.linalg.pinv(a.toarray()) @ vm)) < 1e-8
    assert np.max(np.abs(cols.T @ cols - np.eye(cols.shape[1]))) < 1e-10
    assert np.max(np.abs(cols.T @ np.full(a.n, a.n ** -0.5))) < 1e-10


@pytest.mark.gpu
def test_ritz_values_grow_by_interlacing():
    """test_irlm.py:147-165."""
    a, f, nb = setup(random_connected_graph(30, extra_edges=25, seed=11))
    st = LanczosState(centred_unit(a.n, 5), ncv=12)
    prev = None
    for _ in range(10):
        inverse_lanczos_step(st, a, f, 1e-12, nb)
        mu = np.sort(np.linalg.eigvalsh(st.projected_matrix()))[::-1]
        if prev is not None:
            assert np.all(mu[:prev.shape[0]] >= prev - 1e-12)
        prev = mu


# ---- thick restart (test_irlm.py:168-221) ---------------------------------
def grown(ncv=8):
    a, f, nb = setup(random_connected_graph(30, extra_edges=25, seed=11))
    st = LanczosState(centred_unit(a.n, 5), ncv=ncv)
    while st.m < ncv:
        inverse_lanczos_step(st, a, f, 1e-12, nb)
    return a, f, nb, st


@pytest.mark.gpu
def test_thick_restart_keeps_ritz_values_and_basis():
    """Head = the 3 best Ritz values; 4 orthonormal kernel-free columns
    (test_irlm.py:180-197)."""
    a, f, nb, st = grown()
    mu = np.sort(np.linalg.eigvalsh(st.projected_matrix()))[::-1]
    _thick_restart(st, 2, nb)
    assert st.head_vals.shape == (3,)
    assert np.max(np.abs(st.head_vals - mu[:3])) < 1e-12
    cols = np.column_stack(st.columns)
    assert cols.shape[1] == 4
    assert np.max(np.abs(cols.T @ cols - np.eye(4))) < 1e-10
    assert np.max(np.abs(cols.T @ np.full(a.n, a.n ** -0.5))) < 1e-10


@pytest.mark.gpu
def test_arrowhead_after_growth():
    """test_irlm.py:199-210."""
    a, f, nb, st = grown()
    _thick_restart(st, 2, nb)
    inverse_lanczos_step(st, a, f, 1e-12, nb)
    h = st.projected_matrix()
    k = st.head_vals.shape[0]
    assert h.shape == (k + 1, k + 1)
    assert np.allclose(np.diag(h)[:k], st.head_vals)
    assert np.allclose(h[:k, k], st.head_coupling) and np.allclose(h[k, :k], st.head_coupling)
    assert np.max(np.abs(h[:k, :k] - np.diag(st.head_vals))) == 0.0


@pytest.mark.gpu
def test_restarted_solve_stays_accurate():
    """ncv = 6 forces restarts (test_irlm.py:212-221)."""
    oracle, a = dense_positive_pairs(random_connected_graph(30, extra_edges=25, seed=11), neig=3)
    pairs, rep = irlm_smallest(a, 3, ncv=6, delta=1e-8, seed=0)
    assert rep.config["restarts"] > 0
    assert np.max(np.abs(pairs.positive()[0] - oracle.values) / oracle.values) < 1e-7


# ---- irlm_smallest (test_irlm.py:224-292) ---------------------------------
@pytest.mark.gpu
@pytest.mark.parametrize("graph,neig,delta,expect,tol", [
    (path_graph(3), 1, 1e-6, [1.0], 1e-6),
    (complete_graph(3), 2, 1e-8, [3.0, 3.0], 1e-7),
    (star_graph(3), 2, 1e-8, [1.0, 1.0], 1e-7),
    (cycle_graph(4), 2, 1e-8, [2.0, 2.0], 1e-7),
])
def test_irlm_known_spectra(graph, neig, delta, expect, tol):
    """test_irlm.py:225-255."""
    pairs, rep = irlm_smallest(build_laplacian(graph), neig, delta=delta, seed=0)
    values, vectors, _ = pairs.positive()
    assert values == pytest.approx(expect, abs=tol)
    if neig == 1:
        assert abs(vectors[:, 0] @ V2) == pytest.approx(1.0, abs=1e-6) and rep.converged


@pytest.mark.gpu
def test_irlm_matches_dense_oracle_and_accounting():
    """test_irlm.py:257-277."""
    oracle, a = dense_positive_pairs(random_connected_graph(50, extra_edges=60, seed=7), neig=5)
    pairs, rep = irlm_smallest(a, 5, delta=1e-6, seed=0)
    values, vectors, _ = pairs.positive()
    assert np.max(np.abs(values - oracle.values) / oracle.values) < 1e-5
    _, res = rayleigh_residuals(a, vectors, MvpCounter())
    assert np.max(res) <= 1e-6
    assert pairs.gram_defect() < 1e-8 and pairs.kernel_overlap() < 1e-8
    assert rep.mvp == rep.inner_its_total + rep.config["mvp_verify"]
    assert rep.outer_its > 0
    assert rep.config["delta_pcg"] == pytest.approx(1e-8) and rep.config["ncv"] == 30


@pytest.mark.gpu
def test_irlm_deterministic_and_start_vector():
    """test_irlm.py:279-292 (same seed -> bitwise same; v0 honoured)."""
    a = build_laplacian(random_connected_graph(40, extra_edges=30, seed=3))
    (p1, r1), (p2, r2) = (irlm_smallest(a, 3, delta=1e-6, seed=5) for _ in range(2))
    assert np.array_equal(p1.values, p2.values) and np.array_equal(p1.vectors, p2.vectors)
    assert r1.mvp == r2.mvp
    pairs, rep = irlm_smallest(build_laplacian(path_graph(3)), 1, delta=1e-6,
                               v0=np.array([1.0, 0.0, -1.0]))
    assert pairs.positive()[0][0] == pytest.approx(1.0, abs=1e-6) and rep.converged


@pytest.mark.gpu
def test_irlm_rejects_bad_neig():
    a = build_laplacian(path_graph(3))
    with pytest.raises(ValueError, match="only 2 exist"):
        irlm_smallest(a, 3)
    with pytest.raises(ValueError):
        irlm_smallest(a, 0)
