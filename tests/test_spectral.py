"""spectral.py: Fiedler pair, relaxed cuts, lambda_max, pseudoinverse
approximations, gap diagnostics (the reference's tests/test_spectral.py
cases: P3 / P4 / C4 known answers, dense-eigh agreement, validation).

Host-only helpers and argument validation run on CPU; everything that
touches the operator is @pytest.mark.gpu and goes through the C ABI."""

import math

import numpy as np
import pytest

import paper_1311_1695_b200 as L
from paper_1311_1695_b200.graphs import EdgeList
from paper_1311_1695_b200.spectral import (PinvApprox, cut_weight, estimate_lambda_max,
                                           fiedler, fiedler_order, gap_ratios, make_pinv,
                                           partition_relaxed, pinv_apply, pinv_dense,
                                           sign_partition)


def _dense(a):
    """Dense Laplacian of an EdgeList (D - W) or of a CsrMatrix."""
    if isinstance(a, EdgeList):
        m = np.zeros((a.n_nodes, a.n_nodes))
        m[a.i, a.j] -= a.w
        m[a.j, a.i] -= a.w
        m[np.diag_indices(a.n_nodes)] = -m.sum(axis=1)
        return m
    m = np.zeros((a.n, a.n))
    for r in range(a.n):
        for p in range(a.row_ptr[r], a.row_ptr[r + 1]):
            m[r, a.col_idx[p]] = a.values[p]
    return m


def _csr(g):
    """Host CsrMatrix of an EdgeList's Laplacian (no device needed)."""
    m = _dense(g)
    nz = m != 0
    return L.CsrMatrix(m.shape[0], np.concatenate(([0], np.cumsum(nz.sum(axis=1)))),
                       np.nonzero(nz)[1], m[nz], symmetric=True)


def _pairs(a, k=None):
    """The k smallest positive eigenpairs from a dense eigh (test oracle)."""
    w, v = np.linalg.eigh(_dense(a))
    w, v = w[1:], v[:, 1:]
    if k is not None:
        w, v = w[:k], v[:, :k]
    return L.EigenPairSet(values=w, vectors=v, residuals=np.zeros(w.size))


# ------------------------------------------------------------------ CPU ----

def test_fiedler_order_is_stable_argsort():
    v = np.array([0.5, -1.0, 0.5, 0.0])
    assert fiedler_order(v).tolist() == [1, 3, 0, 2]


def test_partition_relaxed_c4_and_p4():
    a = L.generators.cycle_graph(4)
    x, val = partition_relaxed(_pairs(a), 2, 2)
    assert val == pytest.approx(2.0)              # (n1 n2 / n) * lambda_2 = 1 * 2
    assert x @ _dense(a) @ x == pytest.approx(val)
    assert x @ x == pytest.approx(1.0)            # n / 4
    a = L.generators.path_graph(4)
    x, val = partition_relaxed(_pairs(a), 1, 3)
    assert val == pytest.approx(0.75 * (2 - math.sqrt(2)))
    assert x.sum() == pytest.approx((1 - 3) / 2)  # e'x = (n1 - n2) / 2


def test_split_validation():
    a = L.generators.path_graph(4)
    with pytest.raises(ValueError, match="invalid split"):
        partition_relaxed(_pairs(a), 0, 4)
    with pytest.raises(ValueError, match="invalid split"):
        sign_partition(np.zeros(4), 2, 3)
    with pytest.raises(ValueError, match="lambda_2"):
        partition_relaxed(L.EigenPairSet(np.zeros(0), np.zeros((4, 0)), np.zeros(0)), 2, 2)


def test_sign_partition_and_cut_weight():
    labels = sign_partition(np.array([0.0, 1.0, 0.0, -1.0]), 2, 2)
    assert labels.tolist() == [1, 1, 2, 2]        # tie at 0.0 to the smaller index
    g = L.generators.path_graph(4)
    assert cut_weight(g, np.array([1, 1, 2, 2])) == pytest.approx(1.0)
    g = EdgeList(3, np.array([0, 1]), np.array([1, 2]), np.array([2.0, 5.0]))
    assert cut_weight(g, np.array([1, 2, 2])) == pytest.approx(2.0)


def test_relaxed_value_bounds_every_cut():
    g = L.generators.ba_graph(10, 2, seed=3)
    _, val = partition_relaxed(_pairs(g), 5, 5)
    from itertools import combinations
    best = min(cut_weight(g, np.where(np.isin(np.arange(10), s), 1, 2))
               for s in combinations(range(10), 5))
    assert val <= best + 1e-12


def test_gap_ratios():
    gap, xi = gap_ratios([1.0, 2.0, 4.0])
    assert gap == 4.0 and xi == [1.0, 1.0]
    assert gap_ratios([1.0, 1.0])[1] == [math.inf]
    assert gap_ratios([3.0]) == (1.0, [])
    for bad in ([], [2.0, 1.0], [0.0, 1.0]):
        with pytest.raises(ValueError):
            gap_ratios(bad)


def test_pinv_validation():
    a = L.generators.path_graph(5)
    p = _pairs(a, 2)
    with pytest.raises(ValueError, match="unknown kind"):
        PinvApprox(kind="other", k=1, pairs=p)
    with pytest.raises(ValueError, match="exceeds"):
        PinvApprox(kind="truncated", k=3, pairs=p)
    with pytest.raises(ValueError, match="sigma > 0"):
        PinvApprox(kind="shifted", k=1, pairs=p, sigma=0.0)
    with pytest.raises(ValueError, match="needs the operator"):
        make_pinv(p, 1, kind="shifted", sigma="midpoint")
    with pytest.raises(ValueError, match="unknown sigma policy"):
        make_pinv(p, 1, kind="shifted", sigma="other")
    with pytest.raises(ValueError, match="at least one resolved pair"):
        make_pinv(p, 0, kind="shifted", sigma="lambdak")
    assert make_pinv(p, 2, kind="shifted", sigma="lambdak").sigma == pytest.approx(p.values[1])
    with pytest.raises(ValueError, match="refusing"):
        pinv_dense(make_pinv(p, 1), max_n=4)


def test_fiedler_rejections():
    g = EdgeList(4, np.array([0, 2]), np.array([1, 3]), np.array([1.0, 1.0]))
    with pytest.raises(ValueError, match="2 components"):
        fiedler(_csr(g))
    a = _csr(L.generators.path_graph(3))
    with pytest.raises(ValueError, match="unknown solver"):
        fiedler(a, solver="lobpcg")


# ------------------------------------------------------------------ GPU ----

@pytest.mark.gpu
def test_fiedler_p3_p4_and_solvers_agree():
    a = L.build_laplacian(L.generators.path_graph(3))
    lam, v = fiedler(a, delta=1e-10)
    assert lam == pytest.approx(1.0, abs=1e-9)
    assert abs(v @ np.array([1.0, 0.0, -1.0]) / math.sqrt(2)) == pytest.approx(1.0, abs=1e-8)
    a = L.build_laplacian(L.generators.path_graph(4))
    assert fiedler(a, delta=1e-10)[0] == pytest.approx(2 - math.sqrt(2), abs=1e-9)
    a = L.build_laplacian(L.generators.ba_graph(60, 2, seed=1))
    ref = np.linalg.eigvalsh(_dense(a))[1]
    for s in ("dacg", "jd", "irlm"):
        assert fiedler(a, solver=s, delta=1e-10)[0] == pytest.approx(ref, rel=1e-8)


@pytest.mark.gpu
def test_estimate_lambda_max_and_counter():
    a = L.build_laplacian(L.generators.ba_graph(80, 3, seed=2))
    top = np.linalg.eigvalsh(_dense(a))[-1]
    c = L.MvpCounter()
    est = estimate_lambda_max(a, iters=200, seed=0, counter=c)
    assert c.count == 200
    assert est == pytest.approx(top, rel=1e-3)
    # the reference's recurrence, step for step (same start vector)
    rng = np.random.default_rng(0)
    x = rng.standard_normal(a.n)
    x /= np.linalg.norm(x)
    m = _dense(a)
    for _ in range(20):
        y = m @ x
        th = float(x @ y)
        x = y / np.linalg.norm(y)
    assert estimate_lambda_max(a, seed=0) == pytest.approx(th, rel=1e-12)


@pytest.mark.gpu
def test_pinv_truncated_full_rank_is_pinv():
    a = L.build_laplacian(L.generators.ba_graph(40, 2, seed=4))
    p = make_pinv(_pairs(a), a.n - 1)
    dense = pinv_dense(p)
    assert np.allclose(dense, np.linalg.pinv(_dense(a)), atol=1e-10)


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["truncated", "shifted"])
def test_pinv_apply_matches_formula(kind):
    a = L.build_laplacian(L.generators.ba_graph(300, 3, seed=5))
    pairs = _pairs(a, 6)
    p = make_pinv(pairs, 4, kind=kind, sigma="midpoint", a=a)
    v = np.random.default_rng(7).standard_normal(a.n)
    lam, vk = pairs.values[:4], pairs.vectors[:, :4]
    c = vk.T @ v
    if kind == "truncated":
        ref = vk @ (c / lam)
    else:
        ref = (v - v.sum() / a.n) / p.sigma + vk @ (c * (1 / lam - 1 / p.sigma))
    out = pinv_apply(p, v)
    assert isinstance(out, np.ndarray) and out.shape == (a.n,)
    assert np.allclose(out, ref, rtol=1e-12, atol=1e-13)
    assert np.array_equal(pinv_apply(p, v), out)            # deterministic, reusable
    with pytest.raises(ValueError, match="length"):
        pinv_apply(p, v[:-1])


@pytest.mark.gpu
def test_pinv_zero_pairs_shifted_is_scaled_projector():
    a = L.build_laplacian(L.generators.path_graph(6))
    p = make_pinv(_pairs(a), 0, kind="shifted", sigma=2.0)
    n = a.n
    assert np.allclose(pinv_dense(p), (np.eye(n) - np.ones((n, n)) / n) / 2.0, atol=1e-14)
    assert np.allclose(pinv_dense(make_pinv(_pairs(a), 0)), 0.0)


@pytest.mark.gpu
def test_pinv_shifted_no_worse_than_truncated():
    a = L.build_laplacian(L.generators.ba_graph(50, 2, seed=6))
    pairs = _pairs(a)
    exact = np.linalg.pinv(_dense(a))
    for k in (1, 3, 8):
        t = np.linalg.norm(pinv_dense(make_pinv(pairs, k)) - exact)
        s = np.linalg.norm(pinv_dense(make_pinv(pairs, k, kind="shifted", sigma="midpoint",
                                                a=a)) - exact)
        assert s <= t + 1e-12


@pytest.mark.gpu
@pytest.mark.parametrize("kind", ["truncated", "shifted"])
def test_pinv_apply_many_pairs_chunked(kind):
    """k = 150 > 64: three coefficient / combination passes."""
    a = L.build_laplacian(L.generators.ba_graph(300, 3, seed=8))
    pairs = _pairs(a)
    p = make_pinv(pairs, 150, kind=kind, sigma=3.0)
    v = np.random.default_rng(9).standard_normal(a.n)
    lam, vk = pairs.values[:150], pairs.vectors[:, :150]
    c = vk.T @ v
    ref = vk @ (c / lam) if kind == "truncated" else \
        (v - v.mean()) / 3.0 + vk @ (c * (1 / lam - 1 / 3.0))
    assert np.allclose(pinv_apply(p, v), ref, rtol=1e-11, atol=1e-12)
