"""Restates the reference's pkg/tests/test_pcg.py, test_kernels.py,
test_sparse.py and test_ic0.py against the drop-in: deflation bases, PCG and
the JD correction solve (pcg.py), Gram-Schmidt and the dense eigensolvers
(kernels.py), CsrMatrix / spmv (sparse.py), IC(0) and its shift ladder
(ic0.py).  Plus the preconditioner seams the reference tests only reach
through the solvers: precond_apply / projected_precond_apply
(ic0.py:139-150)."""

import numpy as np
import pytest

from lapeig.generators import grid_graph, path_graph, random_connected_graph
from lapeig.graphs import build_laplacian
from lapeig.ic0 import (Ic0Error, ic0_factorize, identity_factor, precond_apply,
                        projected_precond_apply)
from lapeig.kernels import GramSchmidtBreakdown, dense_sym_eig, mgs_orthonormalize, tridiag_eig
from lapeig.pcg import DeflationBasis, jd_correction_solve, kernel_basis, pcg_solve
from lapeig.sparse import CsrMatrix, MvpCounter, spmv
from tests.ref_suite.conftest import random_spd

gpu = pytest.mark.gpu


def qr_basis(rng, n, k):
    return np.linalg.qr(rng.standard_normal((n, k)))[0]


def csr_of(dense, symmetric=True):
    r, c = np.nonzero(dense)
    return CsrMatrix.from_coo(dense.shape[0], r, c, dense[r, c], symmetric=symmetric)


def op(a):
    return lambda x, cnt: spmv(a, x, cnt)


def p3_matrix():
    """[[2,-1,0],[-1,2,-1],[0,-1,2]] (test_sparse.py:9-17)."""
    return CsrMatrix(3, row_ptr=[0, 2, 5, 7], col_idx=[0, 1, 0, 1, 2, 1, 2],
                     values=[2.0, -1.0, -1.0, 2.0, -1.0, -1.0, 2.0], symmetric=True)


def tridiag(n, diag=2.0, off=-1.0):
    """test_ic0.py:13-22."""
    i = np.arange(n)
    rows = np.concatenate([i, i[:-1], i[1:]])
    cols = np.concatenate([i, i[1:], i[:-1]])
    vals = np.concatenate([np.full(n, diag), np.full(2 * (n - 1), off)])
    return CsrMatrix.from_coo(n, rows, cols, vals, symmetric=True)


def arrow(n):
    """Diagonal 3 + 0.1 i plus a dense last row / column of 0.4: no fill
    (test_ic0.py:25-34)."""
    d = np.diag(3.0 + 0.1 * np.arange(n))
    d[n - 1, :n - 1] = d[:n - 1, n - 1] = 0.4
    return csr_of(d)


# ======================= sparse.py (test_sparse.py) ========================
def test_csr_container_host_contract():
    """toarray / nnz, validation errors, from_coo sorting and duplicates,
    identity, diagonal, row views, symmetry defect, frozen arrays
    (test_sparse.py:20-70); host only."""
    a = p3_matrix()
    assert np.array_equal(a.toarray(), [[2.0, -1, 0], [-1, 2, -1], [0, -1, 2]]) and a.nnz == 7
    for bad in (lambda: CsrMatrix(2, [0, 2, 1], [0, 1, 0], [1.0, 1.0, 1.0]),
                lambda: CsrMatrix(2, [1, 2, 3], [0, 1, 0], [1.0, 1.0, 1.0]),
                lambda: CsrMatrix(2, [0, 1, 2], [0, 2], [1.0, 1.0]),
                lambda: CsrMatrix(2, [0, 1, 2], [0, 1], [1.0]),
                lambda: CsrMatrix.from_coo(2, [0, 0], [1, 1], [1.0, 2.0])):
        with pytest.raises(ValueError):
            bad()
    assert np.array_equal(CsrMatrix.from_coo(2, [1, 0, 1], [1, 0, 0], [3.0, 1.0, 2.0]).toarray(),
                          [[1.0, 0.0], [2.0, 3.0]])
    assert np.array_equal(CsrMatrix.identity(4).toarray(), np.eye(4))
    assert np.array_equal(a.diagonal(), [2.0, 2.0, 2.0])
    cols, vals = a.row(1)
    assert list(cols) == [0, 1, 2] and list(vals) == [-1.0, 2.0, -1.0]
    assert a.symmetry_defect() == 0.0
    assert CsrMatrix.from_coo(2, [0, 1], [1, 0], [1.0, 3.0]).symmetry_defect() == pytest.approx(2.0)
    with pytest.raises(ValueError):
        a.values[0] = 9.0


@gpu
def test_spmv_matches_dense(rng):
    """Random sparse matrices n = 1, 3, 17, 100, 5 vectors each, <= 1e-13
    (test_sparse.py:73-84)."""
    for n in (1, 3, 17, 100):
        dense = rng.standard_normal((n, n))
        dense[rng.random((n, n)) > 0.3] = 0.0
        a = csr_of(dense, symmetric=False)
        for _ in range(5):
            x = rng.standard_normal(n)
            want = dense @ x
            assert np.linalg.norm(spmv(a, x) - want) / max(1.0, np.linalg.norm(want)) <= 1e-13


@gpu
def test_spmv_empty_rows_mismatch_and_counter():
    """test_sparse.py:86-99."""
    a = CsrMatrix.from_coo(3, [0], [2], [5.0])
    assert np.array_equal(spmv(a, np.array([1.0, 1.0, 2.0])), [10.0, 0.0, 0.0])
    with pytest.raises(ValueError):
        spmv(p3_matrix(), np.ones(4))
    c = MvpCounter()
    for _ in range(3):
        spmv(p3_matrix(), np.ones(3), c)
    assert c.count == 3
    c.increment(4)
    assert c.count == 7


# ======================= pcg.py (test_pcg.py) ==============================
def test_deflation_basis_host_contract(rng):
    """Orthonormality check, empty / single, appended, kernel bases
    (test_pcg.py:14-52); host only."""
    with pytest.raises(ValueError):
        DeflationBasis(np.ones((4, 2)))
    e = DeflationBasis.empty(5)
    assert (e.n, e.k) == (5, 0)
    s = DeflationBasis.single(np.array([2.0, 0.0, 0.0]))
    assert s.k == 1 and np.allclose(s.columns[:, 0], [1.0, 0.0, 0.0])
    with pytest.raises(ValueError):
        DeflationBasis.single(np.zeros(3))
    b = DeflationBasis.empty(6)
    assert b.appended(np.eye(6)[2]).k == 1 and b.k == 0
    assert np.allclose(kernel_basis(4).columns[:, 0], 0.5)
    kb = kernel_basis(5, labels=np.array([0, 0, 1, 1, 1]))
    assert kb.k == 2 and kb.columns[0, 1] == 0.0
    assert np.allclose(kb.columns[:2, 0], 2 ** -0.5) and np.allclose(kb.columns[2:, 1], 3 ** -0.5)


@gpu
def test_project_out_removes_span_idempotently(rng):
    """test_pcg.py:28-34."""
    basis = DeflationBasis(qr_basis(rng, 12, 4))
    w = basis.project_out(rng.standard_normal(12))
    assert np.abs(basis.columns.T @ w).max() <= 1e-12
    assert np.allclose(basis.project_out(w), w, atol=1e-14)


@gpu
def test_pcg_matches_dense_solve(rng):
    """test_pcg.py:56-66."""
    for n in (5, 30, 100):
        dense = random_spd(n, rng)
        a = csr_of(dense)
        b = rng.standard_normal(n)
        out = pcg_solve(op(a), None, b, 1e-12, 10 * n)
        want = np.linalg.solve(dense, b)
        assert out.converged
        assert np.linalg.norm(out.solution - want) <= 1e-8 * np.linalg.norm(want)


@gpu
def test_pcg_energy_error_decreases(rng):
    """test_pcg.py:68-83."""
    dense = random_spd(40, rng)
    b = rng.standard_normal(40)
    exact = np.linalg.solve(dense, b)
    errs = []
    pcg_solve(op(csr_of(dense)), None, b, 1e-12, 400,
              callback=lambda x: errs.append(float((x - exact) @ dense @ (x - exact))))
    assert np.all(np.diff(errs) <= 1e-12 * max(1.0, errs[0]))


@gpu
def test_deflated_pcg_stays_in_complement(rng):
    """test_pcg.py:85-101."""
    lap = build_laplacian(random_connected_graph(30, extra_edges=40, seed=2, weighted=True))
    kb = kernel_basis(30)
    b = kb.project_out(rng.standard_normal(30))
    overlaps = []
    out = pcg_solve(op(lap), ic0_factorize(lap), b, 1e-10, 300, deflation=kb,
                    callback=lambda x: overlaps.append(np.abs(kb.columns.T @ x).max()))
    assert out.converged and max(overlaps) <= 1e-9
    assert np.linalg.norm(kb.project_out(spmv(lap, out.solution)) - b) <= 1e-8


@gpu
def test_pcg_zero_rhs_and_indefinite(rng):
    """test_pcg.py:103-127."""
    out = pcg_solve(op(CsrMatrix.identity(4)), None, np.zeros(4), 1e-12, 10)
    assert out.converged and out.iterations == 0 and np.array_equal(out.solution, np.zeros(4))
    dense = random_spd(12, rng)
    vals, vecs = np.linalg.eigh(dense)
    shifted = dense - 0.5 * (vals[1] + vals[2]) * np.eye(12)
    b = vecs[:, 0] + 0.1 * rng.standard_normal(12)
    out = pcg_solve(op(csr_of(shifted)), None, b, 1e-12, 200)
    assert out.indefinite and not out.converged and np.all(np.isfinite(out.solution))


@gpu
def test_correction_solve(rng):
    """The correction is orthogonal to Q = [kernel, u] and nonzero; an exact
    eigenvector still gets a usable fallback (test_pcg.py:130-144)."""
    lap = build_laplacian(random_connected_graph(25, extra_edges=20, seed=6, weighted=True))
    kb = kernel_basis(25)
    u = kb.project_out(rng.standard_normal(25))
    u /= np.linalg.norm(u)
    theta = float(u @ spmv(lap, u))
    q = kb.appended(u)
    s = jd_correction_solve(lap, theta, q, spmv(lap, u) - theta * u, ic0_factorize(lap), 1e-2, 20)
    assert abs(s @ u) <= 1e-9 and np.abs(q.columns.T @ s).max() <= 1e-9
    assert np.linalg.norm(s) > 0
    p3 = build_laplacian(path_graph(3))
    q = kernel_basis(3).appended(np.array([1.0, 0.0, -1.0]) / np.sqrt(2))
    s = jd_correction_solve(p3, 1.0, q, np.array([0.5, -1.0, 0.5]), ic0_factorize(p3), 1e-2, 20)
    assert np.linalg.norm(s) > 0 and np.abs(q.columns.T @ s).max() <= 1e-9


# ======================= kernels.py (test_kernels.py) ======================
@gpu
def test_mgs(rng):
    """Unit, orthogonal, norm = residual norm; breakdown inside the span;
    the second sweep cleans a 1e-9 stray; empty basis normalises
    (test_kernels.py:13-54)."""
    basis = qr_basis(rng, 20, 6)
    u, nrm = mgs_orthonormalize(rng.standard_normal(20), basis)
    assert np.abs(basis.T @ u).max() <= 1e-12
    assert np.linalg.norm(u) == pytest.approx(1.0, abs=1e-13) and nrm > 0
    basis = qr_basis(rng, 15, 4)
    v = rng.standard_normal(15)
    assert mgs_orthonormalize(v, basis)[1] == pytest.approx(
        np.linalg.norm(v - basis @ (basis.T @ v)), rel=1e-10)
    basis = qr_basis(rng, 10, 3)
    with pytest.raises(GramSchmidtBreakdown):
        mgs_orthonormalize(basis @ np.array([0.3, -2.0, 1.1]), basis)
    basis = qr_basis(rng, 30, 10)
    stray = rng.standard_normal(30)
    stray -= basis @ (basis.T @ stray)
    u, _ = mgs_orthonormalize(basis[:, 0] + 1e-9 * stray / np.linalg.norm(stray), basis)
    assert np.abs(basis.T @ u).max() <= 1e-12
    u, nrm = mgs_orthonormalize(np.array([3.0, 4.0]), np.zeros((2, 0)))
    assert np.allclose(u, [0.6, 0.8]) and nrm == pytest.approx(5.0)


def tri(alpha, beta):
    t = np.diag(alpha)
    if len(beta):
        t = t + np.diag(beta, 1) + np.diag(beta, -1)
    return t


def test_tridiag_and_dense_eig(rng):
    """Stencil spectrum {0, 1, 3}; agreement with numpy on random
    tridiagonal / symmetric matrices; 2x2 closed form; multiplicities;
    rejects asymmetric and > 512 (test_kernels.py:57-114); host only."""
    vals, vecs = tridiag_eig(np.array([1.0, 2.0, 1.0]), np.array([-1.0, -1.0]))
    t = tri([1.0, 2.0, 1.0], [-1.0, -1.0])
    assert np.allclose(vals, [0.0, 1.0, 3.0], atol=1e-14)
    assert np.abs(vecs.T @ vecs - np.eye(3)).max() <= 1e-14
    assert np.abs(t @ vecs - vecs * vals).max() <= 1e-13
    for n in (1, 2, 7, 50):
        al, be = rng.standard_normal(n), rng.standard_normal(n - 1) if n > 1 else np.zeros(0)
        vals, vecs = tridiag_eig(al, be)
        want = np.linalg.eigvalsh(tri(al, be))
        assert np.abs(vals - want).max() <= 1e-10 * max(1.0, np.abs(want).max())
        assert np.abs(tri(al, be) @ vecs - vecs * vals).max() <= 1e-10
    vals, vecs = dense_sym_eig(np.array([[2.0, 1.0], [1.0, 2.0]]))
    assert np.allclose(vals, [1.0, 3.0], atol=1e-14)
    w = np.array([1.0, -1.0]) / np.sqrt(2)
    assert min(np.linalg.norm(vecs[:, 0] - w), np.linalg.norm(vecs[:, 0] + w)) <= 1e-14
    for n in (1, 3, 12, 50):
        m = rng.standard_normal((n, n))
        h = 0.5 * (m + m.T)
        vals, vecs = dense_sym_eig(h)
        want = np.linalg.eigvalsh(h)
        sc = max(1.0, np.abs(want).max())
        assert np.abs(vals - want).max() <= 1e-10 * sc
        assert np.abs(vecs.T @ vecs - np.eye(n)).max() <= 1e-12
        assert np.abs(h @ vecs - vecs * vals).max() <= 1e-10 * sc
    for n in (2, 9, 50):
        al, be = rng.standard_normal(n), rng.standard_normal(n - 1)
        vt, _ = tridiag_eig(al, be)
        vd, _ = dense_sym_eig(tri(al, be))
        assert np.abs(vt - vd).max() <= 1e-10 * max(1.0, np.abs(vt).max())
    q = qr_basis(rng, 8, 8)
    h = q @ np.diag([1.0, 1, 1, 2, 2, 5, 5, 5]) @ q.T
    vals, vecs = dense_sym_eig(0.5 * (h + h.T))
    assert np.allclose(vals, [1, 1, 1, 2, 2, 5, 5, 5], atol=1e-12)
    assert np.abs(vecs.T @ vecs - np.eye(8)).max() <= 1e-12
    for bad in (np.array([[1.0, 2.0], [0.0, 1.0]]), np.eye(513)):
        with pytest.raises(ValueError):
            dense_sym_eig(bad)


# ======================= ic0.py (test_ic0.py) ==============================
@gpu
def test_ic0_factor_contract():
    """No-fill matrices factor to the exact Cholesky (tridiagonal 1e-14,
    arrow 1e-13); the factor pattern is the lower triangle; the path
    Laplacian needs a shift; an SPD input succeeds unshifted at attempt 1;
    a zero diagonal is hopeless (test_ic0.py:41-102)."""
    for n in (2, 5, 12, 40):
        f = ic0_factorize(tridiag(n))
        assert f.shift == 0.0
        assert np.abs(f.l.toarray() - np.linalg.cholesky(tridiag(n).toarray())).max() <= 1e-14
    f = ic0_factorize(arrow(9))
    assert np.abs(f.l.toarray() - np.linalg.cholesky(arrow(9).toarray())).max() <= 1e-13
    lap = build_laplacian(random_connected_graph(25, extra_edges=30, seed=5, weighted=True))
    f = ic0_factorize(lap)
    want = {(i, int(c)) for i in range(lap.n) for c in lap.row(i)[0] if c <= i}
    assert {(i, int(c)) for i in range(f.l.n) for c in f.l.row(i)[0]} == want
    f = ic0_factorize(build_laplacian(path_graph(20)))
    assert f.shift > 0.0 and f.attempts >= 2
    f = ic0_factorize(tridiag(8))
    assert (f.shift, f.attempts) == (0.0, 1)
    with pytest.raises(Ic0Error):
        ic0_factorize(CsrMatrix.from_coo(2, [0, 1], [1, 0], [1.0, 1.0], symmetric=True))


@gpu
def test_ic0_apply_inverts_no_fill_matrices(rng):
    """test_ic0.py:52-59, plus the shifted path factor stays finite (:85-88)."""
    for a in (tridiag(15), arrow(11)):
        f = ic0_factorize(a)
        for _ in range(5):
            x = rng.standard_normal(a.n)
            assert np.linalg.norm(f.apply(spmv(a, x)) - x) <= 1e-10 * np.linalg.norm(x)
    f = ic0_factorize(build_laplacian(path_graph(20)))
    assert np.all(np.isfinite(f.apply(np.ones(20))))


@gpu
def test_identity_factor_and_ic0_beats_identity(rng):
    """test_ic0.py:105-120."""
    v = rng.standard_normal(7)
    assert np.array_equal(identity_factor(7).apply(v), v)
    for a in (build_laplacian(grid_graph(8, 8)),
              build_laplacian(random_connected_graph(60, extra_edges=90, seed=3, weighted=True)),
              tridiag(50, diag=2.05)):
        spd = csr_of(a.toarray() + 0.05 * np.eye(a.n))
        b = rng.standard_normal(a.n)
        plain = pcg_solve(op(spd), None, b, 1e-10, 500)
        fancy = pcg_solve(op(spd), ic0_factorize(spd), b, 1e-10, 500)
        assert plain.converged and fancy.converged and fancy.iterations < plain.iterations


@gpu
def test_precond_seams(rng):
    """precond_apply is f.apply (ic0.py:139-141); projected_precond_apply is P M P r for any object with project_out
    (ic0.py:144-150); both against a dense restatement of the factor."""
    lap = build_laplacian(random_connected_graph(40, extra_edges=50, seed=4, weighted=True))
    f = ic0_factorize(lap)
    ld = f.l.toarray()
    r = rng.standard_normal(lap.n)
    mr = np.linalg.solve(ld.T, np.linalg.solve(ld, r))
    assert np.linalg.norm(precond_apply(f, r) - mr) <= 1e-12 * np.linalg.norm(mr)
    q = DeflationBasis(qr_basis(rng, lap.n, 3))
    c = q.columns
    proj = lambda v: v - c @ (c.T @ v)  # noqa: E731
    want = proj(np.linalg.solve(ld.T, np.linalg.solve(ld, proj(r))))
    got = projected_precond_apply(f, q, r)
    assert np.linalg.norm(got - want) <= 1e-12 * np.linalg.norm(want)
    assert np.abs(c.T @ got).max() <= 1e-12
