"""CPU oracle: a numpy restatement of the reference's hot path.

TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
bench.py (its cpu_baseline leg and --impl reference arm) may import this
module, and only as the checker / the timed CPU baseline.  The product
package (paper_1311_1695_b200) never imports it.

It restates, function by function, the algorithm of lapeig 0.1.0
(/root/reference/pkg/src/lapeig) so parity can be checked on the GPU box,
where the reference is absent.  It is pinned against the reference's own
outputs: tests/golden/make_golden.py ran the reference in the build
container and tests/test_oracle_golden.py checks this module against those
fixtures (bit-exact CSR and IC(0) factor, eigenvalues / MVP counts of the
three solvers).

Arithmetic follows the reference's numpy/scipy calls where the order
matters: SpMV per-row sums via np.add.reduceat (sparse.py:135-139), degrees
via np.add.at in edge order (graphs.py:257-258), IC(0) with ascending-column
subtraction (ic0.py:48-78; the C twin oracle/ic0_oracle.c does the same for
large matrices), the IC(0) apply via SuperLU with natural ordering
(ic0.py:36-45).  The dense projected eigenproblems use LAPACK (numpy.eigh)
instead of the reference's own tred2/tql2 (kernels.py:58-226) -- a
roundoff-level difference that the parity tolerances absorb.
"""

import ctypes
import time
from dataclasses import dataclass, field
from pathlib import Path

import numpy as np

# ---------------------------------------------------------------- graphs --


def build_laplacian(n, i, j, w):
    """(row_ptr, col, val) of L = D - A (graphs.py:250-263).

    Degrees accumulate with np.add.at over the i endpoints and then the j
    endpoints, in edge order, from 0.0 -- the reference's summation order.
    """
    i = np.asarray(i, dtype=np.int64)
    j = np.asarray(j, dtype=np.int64)
    w = np.asarray(w, dtype=np.float64)
    deg = np.zeros(n)
    np.add.at(deg, i, w)
    np.add.at(deg, j, w)
    r = np.concatenate([i, j, np.arange(n)])
    c = np.concatenate([j, i, np.arange(n)])
    v = np.concatenate([-w, -w, deg])
    order = np.lexsort((c, r))
    counts = np.bincount(r, minlength=n)
    rp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rp[1:])
    return rp, c[order], v[order]


# ------------------------------------------------------------------ SpMV --


class Csr:
    """Plain CSR triple (int64 row_ptr / col, f64 val)."""

    def __init__(self, n, rp, col, val):
        self.n = int(n)
        self.rp = np.ascontiguousarray(rp, dtype=np.int64)
        self.col = np.ascontiguousarray(col, dtype=np.int64)
        self.val = np.ascontiguousarray(val, dtype=np.float64)
        self.nonempty = np.flatnonzero(np.diff(self.rp) > 0)
        self.count = 0

    @property
    def nnz(self):
        return int(self.rp[-1])

    def dense(self):
        out = np.zeros((self.n, self.n))
        rows = np.repeat(np.arange(self.n), np.diff(self.rp))
        out[rows, self.col] = self.val
        return out


def spmv(a, x):
    """y = A x with the reference's per-row reduceat sums (sparse.py:128-139)."""
    a.count += 1
    y = np.zeros(a.n)
    if a.nonempty.size:
        y[a.nonempty] = np.add.reduceat(a.val * x[a.col], a.rp[a.nonempty])
    return y


# ----------------------------------------------------------------- IC(0) --

_SHIFTS = (1e-8, 1e-6, 1e-4, 1e-3, 1e-2)
_FLOOR = 1e-14


def _lower_split(a):
    rows = np.repeat(np.arange(a.n), np.diff(a.rp))
    low = a.col < rows
    diag = np.zeros(a.n)
    on = a.col == rows
    diag[rows[on]] = a.val[on]
    return rows, low, diag


def _factor_python(a, alpha):
    """One no-fill pass in pure Python (ic0.py:48-78); small matrices."""
    rows, low, diag = _lower_split(a)
    lower = [[] for _ in range(a.n)]
    for r, c, v in zip(rows[low], a.col[low], a.val[low]):
        lower[r].append((int(c), float(v)))
    fac = []          # per row: dict col -> value, insertion ascending
    for i in range(a.n):
        row = {}
        for k, aik in lower[i]:
            s = aik
            rk = fac[k]
            # ascending common columns p < k; both dicts are ascending
            for p in (row if len(row) <= len(rk) else rk):
                if p in row and p in rk and p != k:
                    s -= row[p] * rk[p]
            row[k] = s / rk[k]
        scaled = diag[i] * (1.0 + alpha)
        d = scaled
        for v in row.values():
            d -= v * v
        if d <= _FLOOR * abs(scaled) or d <= 0.0:
            return None
        row[i] = float(np.sqrt(d))
        fac.append(row)
    counts = np.array([len(r) for r in fac], dtype=np.int64)
    lrp = np.zeros(a.n + 1, dtype=np.int64)
    np.cumsum(counts, out=lrp[1:])
    lcol = np.fromiter((c for r in fac for c in r), dtype=np.int64, count=int(lrp[-1]))
    lval = np.fromiter((v for r in fac for v in r.values()), dtype=np.float64, count=int(lrp[-1]))
    return lrp, lcol, lval


_CLIB = None


def _c_oracle():
    """oracle/_build/libic0_oracle.so (built by oracle/Makefile) or None."""
    global _CLIB
    if _CLIB is None:
        path = Path(__file__).resolve().parent / "_build" / "libic0_oracle.so"
        if not path.exists():
            _CLIB = False
        else:
            lib = ctypes.CDLL(str(path))
            lib.ic0_oracle_attempt.restype = ctypes.c_int
            lib.ic0_oracle_attempt.argtypes = [ctypes.c_int64] + [ctypes.c_void_p] * 3 + [
                ctypes.c_double, ctypes.c_void_p]
            _CLIB = lib
    return _CLIB or None


def ic0_factorize(a, shift0=0.0, schedule=_SHIFTS, use_c=None):
    """(lrp, lcol, lval, shift, attempts) per ic0.py:81-116, or raise."""
    _, _, diag = _lower_split(a)
    dmax = float(diag.max()) if a.n else 0.0
    shifts = [float(shift0)] + [s for s in schedule if s > shift0]
    if dmax > 0 and 0.1 * dmax > shifts[-1]:
        shifts.append(0.1 * dmax)
    lib = _c_oracle() if use_c is not False else None
    if use_c is None and a.nnz < 2000:
        lib = None
    for k, alpha in enumerate(shifts, start=1):
        if lib is not None:
            rows = np.repeat(np.arange(a.n), np.diff(a.rp))
            nl = int(np.count_nonzero(a.col < rows)) + a.n
            lval = np.empty(nl)
            ok = lib.ic0_oracle_attempt(a.n, a.rp.ctypes.data, a.col.ctypes.data,
                                        a.val.ctypes.data, alpha, lval.ctypes.data)
            if ok:
                low_or_diag = a.col <= rows
                lrp = np.zeros(a.n + 1, dtype=np.int64)
                np.cumsum(np.bincount(rows[low_or_diag], minlength=a.n), out=lrp[1:])
                return lrp, a.col[low_or_diag].copy(), lval, alpha, k
        else:
            res = _factor_python(a, alpha)
            if res is not None:
                return res + (alpha, k)
    raise RuntimeError("IC(0) breakdown at every shift")


class Ic0:
    """z = (L L^T)^{-1} r through SuperLU with natural ordering (ic0.py:24-45)."""

    def __init__(self, n, lrp, lcol, lval):
        from scipy.sparse import csr_matrix
        from scipy.sparse.linalg import splu
        self.n = n
        lc = csr_matrix((lval, lcol, lrp), shape=(n, n)).tocsc()
        self.lu = splu(lc, permc_spec="NATURAL", diag_pivot_thresh=0.0)

    def apply(self, r):
        return self.lu.solve(self.lu.solve(np.asarray(r, dtype=np.float64), trans="N"),
                             trans="T")


class Identity:
    def apply(self, r):
        return np.array(r, dtype=np.float64)


# ------------------------------------------------------------ projections --


def project(c, v):
    """v - C (C^T v); a fresh copy when C has no columns (pcg.py:55-60)."""
    if c.shape[1] == 0:
        return np.array(v, dtype=np.float64)
    return v - c @ (c.T @ v)


def kernel_columns(n):
    return np.full((n, 1), 1.0 / np.sqrt(n))


def gram_schmidt(v, basis):
    """MGS with one conditional second sweep (kernels.py:22-55)."""
    v = np.array(v, dtype=np.float64)
    if basis.ndim == 1:
        basis = basis.reshape(-1, 1)
    nin = np.linalg.norm(v)
    if nin == 0.0:
        raise ArithmeticError("zero vector")
    k = basis.shape[1] if basis.size else 0
    prev = nin
    for _sweep in range(2):
        for col in range(k):
            q = basis[:, col]
            v -= (q @ v) * q
        now = np.linalg.norm(v)
        if k == 0 or now >= 0.7 * prev:
            break
        prev = now
    nout = np.linalg.norm(v)
    if nout < 1e-14 * nin:
        raise ArithmeticError("Gram-Schmidt breakdown")
    return v / nout, nout


# -------------------------------------------------------------------- PCG --


@dataclass
class PcgResult:
    x: np.ndarray
    its: int
    relres: float
    converged: bool
    indefinite: bool = False


def pcg(op, prec, b, tol, maxit, c=None):
    """Deflated PCG (pcg.py:96-156): residual and preconditioned residual
    stay projected; nonpositive curvature stops the iteration."""
    proj = (lambda v: v) if c is None or c.shape[1] == 0 else (lambda v: project(c, v))
    bh = np.array(b, dtype=np.float64) if c is None or c.shape[1] == 0 else proj(b)
    nb = np.linalg.norm(bh)
    if nb == 0.0:
        return PcgResult(np.zeros_like(bh), 0, 0.0, True)
    x = np.zeros_like(bh)
    r = bh.copy()
    z = proj(prec(r))
    rz = r @ z
    p = z.copy()
    rel, it = 1.0, 0
    while it < maxit:
        ap = proj(op(p))
        it += 1
        pap = p @ ap
        if pap <= 0.0:
            return PcgResult(x, it, rel, False, True)
        g = rz / pap
        x += g * p
        r -= g * ap
        r = proj(r)
        rel = np.linalg.norm(r) / nb
        if rel <= tol:
            return PcgResult(x, it, rel, True)
        z = proj(prec(r))
        rz2 = r @ z
        if rz2 <= 0.0:
            return PcgResult(x, it, rel, False, True)
        p = z + (rz2 / rz) * p
        rz = rz2
    return PcgResult(x, it, rel, False)


# ------------------------------------------------------------------- DACG --


@dataclass
class Result:
    values: np.ndarray
    vectors: np.ndarray
    residuals: np.ndarray
    mvp: int
    outer: int = 0
    inner: int = 0
    wall: float = 0.0
    extra: dict = field(default_factory=dict)


def _plane(x, ax, p, ap):
    """Rayleigh-Ritz on span{x, p} (dacg.py:55-96) -> (mu, alpha, beta)."""
    sx = np.linalg.norm(x)
    sp = np.linalg.norm(p)
    if sx == 0.0 or sp == 0.0:
        raise ValueError("degenerate plane")
    xb, axb = x / sx, ax / sx
    cp = xb @ p
    pt = p - cp * xb
    spt = np.linalg.norm(pt)
    if spt <= np.sqrt(1e-12) * sp:
        raise ValueError("degenerate plane")
    pb, apb = pt / spt, (ap - cp * axb) / spt
    h11, h22 = xb @ axb, pb @ apb
    h12 = 0.5 * (xb @ apb + pb @ axb)
    mu = 0.5 * (h11 + h22) - np.hypot(0.5 * (h11 - h22), h12)
    ra, rb = (h11 - mu, h12), (h12, h22 - mu)
    row = ra if np.hypot(*ra) >= np.hypot(*rb) else rb
    u, v = row[1], -row[0]
    nr = np.hypot(u, v)
    if nr == 0.0:
        u, v, nr = 1.0, 0.0, 1.0
    u, v = u / nr, v / nr
    al = u / sx - v * cp / (spt * sx)
    be = v / spt
    sc = np.hypot(al, be)
    return mu, al / sc, be / sc


def dacg(a, neig, delta=1e-6, f=None, maxit=20000, seed=0, null=None, deadline=None):
    """DACG (dacg.py:122-276) with the same RNG stream and acceptance test."""
    t0 = time.perf_counter()
    a.count = 0
    n = a.n
    guard = kernel_columns(n) if null is None else null
    rng = np.random.default_rng(seed)
    reset = max(1, n // 10)
    vals, vecs, res_out, its = [], [], [], []
    for pair in range(neig):
        x = project(guard, rng.standard_normal(n))
        x /= np.linalg.norm(x)
        ax = spmv(a, x)
        q = x @ ax
        g = 2.0 * (ax - q * x)
        pdir = None
        gprev = zprev = None
        since = 0
        k = 0
        done = None
        while k < maxit:
            if deadline is not None and time.perf_counter() > deadline:
                raise TimeoutError(k)
            rs = np.linalg.norm(ax - q * x)
            if q > 0 and rs / q <= delta:
                xc = project(guard, x)
                xc /= np.linalg.norm(xc)
                wv = spmv(a, xc)
                th = xc @ wv
                rf = np.linalg.norm(wv - th * xc)
                if th > 0 and rf / th <= delta:
                    done = (th, xc, rf / th)
                    break
                x, ax, q = xc, wv, th
                g = 2.0 * (wv - th * xc)
            z = project(guard, f.apply(g))
            if gprev is None or since >= reset:
                beta, since = 0.0, 0
            else:
                den = gprev @ zprev
                beta = ((g - gprev) @ z) / den if den != 0 else 0.0
                beta = max(beta, 0.0)
            p = -z + beta * pdir if (beta != 0.0 and pdir is not None) else -z
            p = project(guard, p)
            p -= (x @ p) * x
            tries = 0
            while True:
                bxx, bpp, bxp = x @ x, p @ p, x @ p
                if not (bpp == 0.0 or bxx * bpp - bxp * bxp <= 1e-12 * bxx * bpp):
                    break
                tries += 1
                if tries > 3:
                    raise RuntimeError("no search direction")
                p = project(guard, -z if tries == 1 else rng.standard_normal(n))
                p -= (x @ p) * x
            ap = spmv(a, p)
            mu, al, be = _plane(x, ax, p, ap)
            xn, axn = al * x + be * p, al * ax + be * ap
            nr = np.linalg.norm(xn)
            xn, axn = xn / nr, axn / nr
            qn = xn @ axn
            if qn > q + 1e-14 * max(1.0, abs(q)):
                raise RuntimeError("Rayleigh quotient increased")
            gprev, zprev = g, z
            x, ax, q = xn, axn, qn
            g = 2.0 * (axn - qn * xn)
            pdir = p
            k += 1
            since += 1
        if done is None:
            raise RuntimeError(f"pair {pair}: iteration cap")
        vals.append(done[0])
        vecs.append(done[1])
        res_out.append(done[2])
        its.append(k)
        guard = np.hstack([guard, done[1].reshape(-1, 1)])
    order = np.argsort(vals, kind="stable")
    return Result(np.asarray(vals)[order], np.column_stack(vecs)[:, order],
                  np.asarray(res_out)[order], a.count, 0, int(sum(its)),
                  time.perf_counter() - t0, {"iterations_per_pair": its})


# --------------------------------------------------------------------- JD --


def _small_eig(h):
    w, v = np.linalg.eigh(0.5 * (h + h.T))
    return w, v


def jd(a, neig, delta=1e-6, delta_pcg=1e-2, itmax=20, m_min=5, m_max=10, f=None, seed=0,
       max_outer=300, stagnation=60, null=None, deadline=None):
    """Jacobi-Davidson (jd.py:100-255) with the projected PCG correction
    solve (pcg.py:159-184)."""
    t0 = time.perf_counter()
    a.count = 0
    n = a.n
    guard = kernel_columns(n) if null is None else null
    rng = np.random.default_rng(seed)
    V = np.zeros((n, 0))
    W = np.zeros((n, 0))
    H = np.zeros((0, 0))
    cand = rng.standard_normal(n)
    locked, lvecs, lres = [], [], []
    best, since, here = np.inf, 0, 0
    outer = inner = restarts = 0
    while len(locked) < neig:
        if deadline is not None and time.perf_counter() > deadline:
            raise TimeoutError(outer)
        here += 1
        if here > max_outer:
            raise RuntimeError("outer cap")
        full = guard.shape[1] + V.shape[1] >= n
        if not full:
            blk = np.hstack([guard, V])
            try:
                v, _ = gram_schmidt(cand, blk)
            except ArithmeticError:
                v, _ = gram_schmidt(rng.standard_normal(n), blk)
            w = spmv(a, v)
            m = V.shape[1]
            Hn = np.zeros((m + 1, m + 1))
            Hn[:m, :m] = H
            Hn[:m, m] = V.T @ w
            Hn[m, :m] = v @ W
            Hn[m, m] = v @ w
            H = 0.5 * (Hn + Hn.T)
            V = np.hstack([V, v.reshape(-1, 1)])
            W = np.hstack([W, w.reshape(-1, 1)])
        th, y = _small_eig(H)
        theta, yy = th[0], y[:, 0]
        u = V @ yy
        nu = np.linalg.norm(u)
        u /= nu
        r = W @ yy / nu - theta * u
        if theta <= 0:
            raise RuntimeError("nonpositive Ritz value")
        rn = np.linalg.norm(r)
        if rn < best * (1 - 1e-3):
            best, since = rn, 0
        else:
            since += 1
        if rn < delta * theta:
            uf, _ = gram_schmidt(u, guard)
            wf = spmv(a, uf)
            tf = uf @ wf
            rf = np.linalg.norm(wf - tf * uf)
            if rf < delta * tf:
                locked.append(tf)
                lvecs.append(uf)
                lres.append(rf / tf)
                guard = np.hstack([guard, uf.reshape(-1, 1)])
                best, since, here = np.inf, 0, 0
                th, y = _small_eig(H)
                V, W = V @ y[:, 1:], W @ y[:, 1:]
                H = np.diag(th[1:])
                cand = rng.standard_normal(n)
                continue
        if full:
            raise RuntimeError("space exhausted")
        if since > stagnation:
            raise RuntimeError("stagnation")
        if V.shape[1] == m_max:
            th, y = _small_eig(H)
            keep = y[:, :m_min]
            V, W = V @ keep, W @ keep
            H = np.diag(th[:m_min])
            qv, _ = np.linalg.qr(V)
            sg = np.sign(np.einsum("ij,ij->j", qv, V))
            sg[sg == 0] = 1.0
            V = qv * sg
            restarts += 1
        Q = np.hstack([guard, (u / np.linalg.norm(u)).reshape(-1, 1)])
        before = a.count

        def op(x, Q=Q, theta=theta):
            return project(Q, spmv(a, x) - theta * x)

        prec = (lambda rr, Q=Q: project(Q, f.apply(project(Q, rr)))) if f is not None else None
        out = pcg(op, prec if prec else (lambda rr: rr), -r, delta_pcg, itmax, Q)
        s = out.x
        if np.linalg.norm(s) == 0.0 and np.linalg.norm(r) > 0.0:
            s = project(Q, f.apply(project(Q, -r))) if f is not None else project(Q, -r)
        cand = s
        outer += 1
        inner += a.count - before
    order = np.argsort(locked, kind="stable")
    return Result(np.asarray(locked)[order], np.column_stack(lvecs)[:, order],
                  np.asarray(lres)[order], a.count, outer, inner,
                  time.perf_counter() - t0, {"restarts": restarts})


# ------------------------------------------------------------------- IRLM --


def ncv_for(neig):
    """Subspace size schedule (irlm.py:24-37)."""
    pts = ((1, 15), (5, 30), (20, 60), (50, 120))
    if neig <= 1:
        return 15
    for (x0, y0), (x1, y1) in zip(pts, pts[1:]):
        if neig <= x1:
            return int(round(y0 + (y1 - y0) * (neig - x0) / (x1 - x0)))
    return 120 + 2 * (neig - 50)


def irlm(a, neig, delta=1e-6, f=None, seed=0, ncv=None, maxit_inner=5000, max_restarts=200,
         null=None, deadline=None):
    """Inverse Lanczos with thick restart (irlm.py:230-321)."""
    t0 = time.perf_counter()
    a.count = 0
    n = a.n
    null = kernel_columns(n) if null is None else null
    usable = n - null.shape[1]
    ncv = min(max(ncv_for(neig) if ncv is None else ncv, neig + 2), usable)
    dpcg = 1e-2 * delta
    rng = np.random.default_rng(seed)
    v1, _ = gram_schmidt(rng.standard_normal(n), null)
    cols = [v1]
    head = np.zeros(0)
    coup = np.zeros(0)
    alpha, beta = [], []
    broke = False
    solves = inner = 0

    def dim():
        return head.size + len(alpha)

    def proj_matrix():
        k, t = head.size, len(alpha)
        h = np.zeros((k + t, k + t))
        h[np.arange(k), np.arange(k)] = head
        if k and t:
            h[:k, k] = coup
            h[k, :k] = coup
        for s in range(t):
            h[k + s, k + s] = alpha[s]
            if s + 1 < t:
                h[k + s, k + s + 1] = h[k + s + 1, k + s] = beta[s]
        return h

    def ritz():
        mu, y = np.linalg.eigh(proj_matrix())
        o = np.argsort(mu, kind="stable")[::-1]
        return mu[o], y[:, o]

    def check():
        m = dim()
        if m < neig:
            return None
        _, y = ritz()
        V = np.column_stack(cols[:m])
        th = np.zeros(neig)
        rs = np.zeros(neig)
        U = np.zeros((n, neig))
        for i in range(neig):
            u = V @ y[:, i]
            u /= np.linalg.norm(u)
            w = spmv(a, u)
            t = u @ w
            if t <= 0:
                return None
            rr = np.linalg.norm(w - t * u) / t
            if rr > delta:
                return None
            th[i], rs[i], U[:, i] = t, rr, u
        if rs.mean() > delta:
            return None
        o = np.argsort(th, kind="stable")
        return th[o], U[:, o], rs[o]

    result = None
    for cycle in range(max_restarts + 1):
        while dim() < ncv and not broke:
            if deadline is not None and time.perf_counter() > deadline:
                raise TimeoutError(solves)
            v = cols[-1]
            out = pcg(lambda x: spmv(a, x), f.apply, v, dpcg, maxit_inner, null)
            if not out.converged:
                raise RuntimeError("inner PCG stalled")
            inner += out.its
            solves += 1
            w = out.x
            scale = max(1.0, np.linalg.norm(w))
            al = w @ v
            w = w - al * v
            if not alpha:
                if head.size:
                    w -= np.column_stack(cols[:head.size]) @ coup
            else:
                w -= beta[-1] * cols[-2]
            for _ in range(2):
                w = project(null, w)
                for c in cols:
                    w -= (c @ w) * c
            b = np.linalg.norm(w)
            alpha.append(al)
            if b < 1e-12 * scale:
                broke = True
            else:
                beta.append(b)
                cols.append(w / b)
        if broke:
            ins = False
            for _ in range(3):
                try:
                    v, _ = gram_schmidt(rng.standard_normal(n), np.column_stack([null] + cols))
                except ArithmeticError:
                    continue
                beta.append(0.0)
                cols.append(v)
                broke = False
                ins = True
                break
            if ins:
                continue
            result = check()
            if result is None:
                raise RuntimeError("subspace exhausted")
            break
        result = check()
        if result is not None:
            break
        if cycle == max_restarts:
            raise RuntimeError("no convergence")
        m = dim()
        keep = min(neig + 1, m - 1)
        mu, y = ritz()
        V = np.column_stack(cols[:m])
        heads = V @ y[:, :keep]
        new = []
        for s in range(keep):
            blk = np.column_stack([null] + new) if (null.shape[1] or new) else np.zeros((n, 0))
            vv, _ = gram_schmidt(heads[:, s], blk)
            new.append(vv)
        res = project(null, cols[-1])
        for c in new:
            res -= (c @ res) * c
        res /= np.linalg.norm(res)
        coup = beta[-1] * y[m - 1, :keep]
        head = mu[:keep].copy()
        cols = new + [res]
        alpha, beta = [], []
    vals, vecs, rs = result
    return Result(vals, vecs, rs, a.count, solves, inner, time.perf_counter() - t0)


def rayleigh_residuals(a, vectors):
    """Independent residual recomputation (results.py:90-105)."""
    vectors = np.asarray(vectors, dtype=np.float64).reshape(a.n, -1)
    th = np.zeros(vectors.shape[1])
    rs = np.zeros(vectors.shape[1])
    for k in range(vectors.shape[1]):
        u = vectors[:, k]
        w = spmv(a, u)
        nn = u @ u
        t = (u @ w) / nn
        d = abs(t) if t != 0 else 1.0
        rs[k] = np.linalg.norm(w - t * u) / (np.sqrt(nn) * d)
        th[k] = t
    return th, rs
