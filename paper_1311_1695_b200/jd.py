"""Jacobi-Davidson with sequential deflation, on the B200.

Mirrors the reference module jd.py (lapeig 0.1.0):

    JdWorkspace             jd.py:21-57   search basis V, image W = A V, H = V'AV
    rayleigh_ritz_extract   jd.py:60-76
    jd_restart              jd.py:79-97
    jd_smallest             jd.py:100-255 same signature, RNG stream, locking,
                                          stagnation and saturation logic

Device layout: one (kcap, n) column block B holds [locked guard | V]
contiguously (rows = columns), so Gram-Schmidt against hstack[guard, V]
(jd.py:157) is a single block projection; W is an (m_max, n) block.  The
projected matrix H (at most m_max x m_max) and its eigenproblem stay on the
host.  The correction equation runs on DevicePcg (pcg.py); its projection
basis [guard | u] is passed as two blocks, never copied.
"""

import time

import numpy as np

from . import _device as dev
from ._plan import Ctx, Fused, Slots
from ._rng import NormalStream
from .ic0 import ic0_factorize
from .kernels import DeviceGS, GramSchmidtBreakdown, dense_sym_eig
from .pcg import DevicePcg, kernel_basis
from .precond import device_preconditioner
from .results import EigenPairSet, SolverError, SolverReport
from .sparse import MvpCounter, device_csr


class JdWorkspace:
    """Search basis V, its image W = A V and projected matrix H = V'AV.

    Vectors are kept on the device ((m_max, n) blocks); .v / .w return host
    copies in the reference's (n, m) layout.
    """

    def __init__(self, n, m_min, m_max):
        if not 0 < m_min < m_max:
            raise ValueError("need 0 < m_min < m_max")
        self.n = int(n)
        self.m_min = int(m_min)
        self.m_max = int(m_max)
        self.V = dev.zeros((self.m_max + 1, self.n))
        self.W = dev.zeros((self.m_max + 1, self.n))
        self._m = 0
        self.h = np.zeros((0, 0))
        self.theta = None
        self.u = None
        self.S = Slots(capacity=256)
        self.S.add("d", 2 * self.m_max + 8)

    @property
    def m(self):
        return self._m

    @property
    def v(self):
        return dev.to_host(self.V[:self._m]).T.copy()

    @v.setter
    def v(self, value):
        self._set_block(self.V, value)

    @property
    def w(self):
        return dev.to_host(self.W[:self._m]).T.copy()

    @w.setter
    def w(self, value):
        self._set_block(self.W, value)

    def _set_block(self, blk, value):
        arr = np.asarray(dev.to_host(value), dtype=np.float64).reshape(self.n, -1)
        m = arr.shape[1]
        if m > self.m_max + 1:
            raise ValueError("block wider than m_max")
        blk[:m] = dev.to_device(np.ascontiguousarray(arr.T))
        self._m = m

    def append(self, v_new, w_new):
        """Grow the basis by an orthonormal column and its image; H gains
        the bordered row/column and is symmetrized (jd.py:39-57)."""
        m = self._m
        if m >= self.m_max + 1:
            raise ValueError("workspace is full")
        self.V[m] = dev.to_device(v_new)
        self.W[m] = dev.to_device(w_new)
        S = self.S
        # col = V^T w_new (m), diag = v_new.w_new; row = v_new^T W (m)
        Fused(self.n, blocks=[(self.V, m + 1, self.W[m]), (self.W, m, self.V[m])],
              result=S.s[S.idx["d"]:])()
        s = S.fetch()[0][S.idx["d"]:S.idx["d"] + 2 * m + 1]
        col, diag, row = s[:m], s[m], s[m + 1:2 * m + 1]
        h = np.zeros((m + 1, m + 1))
        h[:m, :m] = self.h
        h[:m, m] = col
        h[m, :m] = row
        h[m, m] = diag
        self.h = 0.5 * (h + h.T)
        self._m = m + 1


def _ritz(ws, S, u_out, r_out, cx=None):
    """theta, and on the device u = Vy/|Vy|, r = (Wy - theta Vy)/|Vy|;
    returns (theta, |r|^2)."""
    cx = cx or Ctx(ws.n)
    vals, vecs = dense_sym_eig(ws.h)
    y = vecs[:, 0]
    theta = float(vals[0])
    m = ws.m
    S.set_vec("y", y)
    S.set(theta=theta)
    n = ws.n
    # u_raw = V y, wy = W y (block updates with cscale -1), |u_raw|^2
    cx.fused(outs=[dict(out=ws._ur, terms=[], upd=(ws.V, m, S.p("y"), -1.0)),
                   dict(out=ws._wy, terms=[], upd=(ws.W, m, S.p("y"), -1.0))],
          dots=[(1, None)], result=S.s[S.idx["nu2"]:])()
    cx.fused(outs=[dict(out=u_out, terms=[(ws._ur, 1.0)], post=(S.p("nu2"), 3)),
                   dict(out=r_out, terms=[(ws._wy, 1.0), (ws._ur, -1.0, S.p("theta"))],
                        post=(S.p("nu2"), 3))],
          dots=[(2, None)], result=S.s[S.idx["rr"]:])()
    rr = float(S.fetch()[0][S.idx["rr"]])
    return theta, rr, vals, vecs


def _ensure_tmp(ws):
    if not hasattr(ws, "_ur"):
        ws._ur = dev.empty(ws.n)
        ws._wy = dev.empty(ws.n)
        for nm, c in (("y", ws.m_max + 1), ("theta", 1), ("nu2", 1), ("rr", 1)):
            ws.S.add(nm, c)


def rayleigh_ritz_extract(workspace):
    """Smallest Ritz pair of the current search space (jd.py:60-76); the
    residual is assembled from W, no product with A."""
    _ensure_tmp(workspace)
    u = dev.empty(workspace.n)
    r = dev.empty(workspace.n)
    theta, _, _, _ = _ritz(workspace, workspace.S, u, r)
    workspace.theta = theta
    workspace.u = dev.to_host(u)
    return theta, workspace.u, dev.to_host(r)


def _gemm(n, src, mrows, ycols, out, cx=None):
    """out[:p] = (src[:mrows] as columns) @ ycols on the device (over this
    rank's rows when cx is row-partitioned)."""
    from . import _native as nat
    yc = np.asfortranarray(np.asarray(ycols, dtype=np.float64))
    lo, nl = (cx.lo, cx.nl) if cx is not None else (0, n)
    nat.call("lg_gemm_small", nl, src.data_ptr() + 8 * lo, n, mrows, yc.ctypes.data,
             yc.shape[1], out.data_ptr() + 8 * lo, n, dev.stream_ptr())


def jd_restart(workspace):
    """Contract the basis to the m_min best Ritz vectors (jd.py:79-97); V is
    re-orthonormalised (Gram-Schmidt QR, positive R diagonal = the
    reference's sign fix), W follows V keep."""
    ws = workspace
    if ws.m <= ws.m_min:
        raise SolverError("restart called below the retention size")
    vals, vecs = dense_sym_eig(ws.h)
    keep = vecs[:, :ws.m_min]
    tv = dev.empty((ws.m_min, ws.n))
    tw = dev.empty((ws.m_min, ws.n))
    _gemm(ws.n, ws.V, ws.m, keep, tv)
    _gemm(ws.n, ws.W, ws.m, keep, tw)
    gs = DeviceGS(ws.n)
    for j in range(ws.m_min):
        gs.run(tv[j], [(ws.V, j)] if j else [], ws.V[j])
    ws.W[:ws.m_min] = tw
    ws.h = np.diag(vals[:ws.m_min])
    ws._m = ws.m_min
    return ws


def jd_smallest(a, neig, delta=1e-6, delta_pcg=1e-2, itmax_inner=20,
                m_min=5, m_max=10, f=None, null_basis=None, *, seed=0,
                max_outer_per_pair=300, stagnation_window=60,
                counter=None, v0=None, comm=None):
    """neig smallest strictly positive eigenpairs of a by Jacobi-Davidson
    (jd.py:100-255).  The outer iteration for a pair stops once
    ||r|| < delta * theta, after which the pair is verified with a fresh
    product and locked; the correction equation runs at relative tolerance
    delta_pcg with at most itmax_inner PCG iterations.

    comm (extension, not in the reference): a dist.RowComm -- one rank of a
    row-partitioned solve, as for dacg_smallest."""
    with dev.solver_stream():
        return _jd_smallest_impl(**locals())


def _jd_smallest_impl(a, neig, delta=1e-6, delta_pcg=1e-2, itmax_inner=20,
                m_min=5, m_max=10, f=None, null_basis=None, *, seed=0,
                max_outer_per_pair=300, stagnation_window=60,
                counter=None, v0=None, comm=None):
    t0 = time.perf_counter()
    if counter is None:
        counter = MvpCounter()
    if null_basis is None:
        null_basis = kernel_basis(a.n)
    dist = comm is not None and comm.world > 1
    if comm is not None and comm.world == 1 and isinstance(f, str):
        # one rank: block-Jacobi IC(0) with one block is the reference IC(0)
        from .precond import FsaiFactor, JacobiFactor
        f = {"jacobi": JacobiFactor, "fsai": FsaiFactor}.get(f, lambda _: None)(a)
    if f is None and not dist:
        f = ic0_factorize(a)
    if neig < 1:
        raise ValueError("neig must be at least 1")
    usable = a.n - null_basis.k
    if neig > usable:
        raise ValueError(f"asked for {neig} pairs but only {usable} exist "
                         "outside the kernel")
    if not 0 < m_min < m_max:
        raise ValueError("need 0 < m_min < m_max")
    rng = np.random.default_rng(seed)
    n = a.n
    draws = NormalStream(rng, n)
    cx = Ctx(n, comm)
    if dist:
        csr = comm.solver_operator(a)
        prec = comm.local_preconditioner(a, f)
    else:
        csr = device_csr(a)
        prec = device_preconditioner(f, n)
    kg = null_basis.k
    kcap = kg + neig + m_max + 1
    if kcap > 64:
        raise ValueError("guard + search space wider than 64 columns")
    B = dev.zeros((kcap, n))
    if kg:
        B[:kg] = null_basis.device()
    W = dev.zeros((m_max + 1, n))
    S = Slots(capacity=512)
    for nm, c in (("y", m_max + 1), ("theta", 1), ("nu2", 1), ("rr", 1), ("hd", 2 * m_max + 4),
                  ("vf", 4)):
        S.add(nm, c)
    gs = DeviceGS(n, cx=cx)
    engine = DevicePcg(csr, prec, n, "jd", kg + neig + 1, cx=cx)
    u = dev.empty(n)
    r = dev.empty(n)
    ufix = dev.empty(n)
    wfix = dev.empty(n)
    tmpv = dev.empty((m_max + 1, n))
    tmpw = dev.empty((m_max + 1, n))
    cand = dev.to_device(v0 if v0 is not None else draws.draw())

    class _Space:  # view of B[kg:kg+m] / W as a workspace for _ritz
        pass

    sp = _Space()
    sp.n, sp.m_max, sp.m_min = n, m_max, m_min
    sp._ur, sp._wy = dev.empty(n), dev.empty(n)
    m = 0
    H = np.zeros((0, 0))

    locked_vals, locked_vecs, locked_res = [], [], []
    outer_solves = inner_total = outer_mvps = verify_mvps = restarts = 0
    best_res, since_best, outer_here = np.inf, 0, 0

    def gemm(src, mrows, ycols, out):
        _gemm(n, src, mrows, ycols, out, cx)

    while len(locked_vals) < neig:
        pair_idx = len(locked_vals)
        outer_here += 1
        if outer_here > max_outer_per_pair:
            raise SolverError(
                f"pair {pair_idx}: no convergence within "
                f"{max_outer_per_pair} outer iterations "
                f"(best residual {best_res:.3e})")
        saturated = kg + m >= n
        if not saturated:
            try:
                gs.run(cand, [(B, kg + m)], B[kg + m])
            except GramSchmidtBreakdown:
                cand = dev.to_device(draws.draw())
                try:
                    gs.run(cand, [(B, kg + m)], B[kg + m])
                except GramSchmidtBreakdown as exc:
                    raise SolverError(
                        f"pair {pair_idx}: search space saturated the "
                        "complement without meeting the tolerance") from exc
            # w_new = A v_new with the epilogue col/diag = V'^T w_new
            cx.spmv(csr, B[kg + m], W[m], q=B[kg:], nq=m + 1, result=S.s[S.idx["hd"]:])()
            counter.increment()
            outer_mvps += 1
            if m:
                cx.fused(blocks=[(W, m, B[kg + m])], result=S.s[S.idx["hd"] + m + 1:])()
            hd = S.fetch()[0][S.idx["hd"]:S.idx["hd"] + 2 * m + 1]
            Hn = np.zeros((m + 1, m + 1))
            Hn[:m, :m] = H
            Hn[:m, m] = hd[:m]
            Hn[m, :m] = hd[m + 1:2 * m + 1]
            Hn[m, m] = hd[m]
            H = 0.5 * (Hn + Hn.T)
            m += 1
        sp.V, sp.W, sp.h, sp.m = B[kg:], W, H, m
        theta, rr, hvals, hvecs = _ritz(sp, S, u, r, cx)
        if theta <= 0:
            raise SolverError(f"pair {pair_idx}: nonpositive Ritz value {theta}")
        res = float(np.sqrt(rr))
        if res < best_res * (1 - 1e-3):
            best_res = res
            since_best = 0
        else:
            since_best += 1
        if res < delta * theta:
            gs.run(u, [(B, kg)], ufix)
            cx.spmv(csr, ufix, wfix, dots=[ufix], result=S.s[S.idx["vf"]:])()
            counter.increment()
            verify_mvps += 1
            theta_fix = float(S.fetch()[0][S.idx["vf"]])
            S.set(theta=theta_fix)
            cx.fused(outs=[dict(out=r, terms=[(wfix, 1.0), (ufix, -1.0, S.p("theta"))])],
                  dots=[(1, None)], result=S.s[S.idx["vf"] + 1:])()
            res_fix = float(np.sqrt(S.fetch()[0][S.idx["vf"] + 1]))
            if res_fix < delta * theta_fix:
                locked_vals.append(theta_fix)
                locked_vecs.append(kg)   # row of B holding the locked vector
                locked_res.append(res_fix / theta_fix)
                # carry the other Ritz directions (jd.py:197-205)
                if m > 1:
                    gemm(B[kg:], m, hvecs[:, 1:], tmpv)
                    gemm(W, m, hvecs[:, 1:], tmpw)
                B[kg] = ufix
                kg += 1
                m -= 1
                if m:
                    B[kg:kg + m] = tmpv[:m]
                    W[:m] = tmpw[:m]
                H = np.diag(hvals[1:])
                best_res, since_best, outer_here = np.inf, 0, 0
                cand = dev.to_device(draws.draw())
                continue
        if saturated:
            raise SolverError(
                f"pair {pair_idx}: exhausted the whole space at residual "
                f"{res:.3e} (target {delta * theta:.3e})")
        if since_best > stagnation_window:
            raise SolverError(
                f"pair {pair_idx}: stagnated for {since_best} outer "
                f"iterations at residual {best_res:.3e} "
                f"(target {delta * theta:.3e})")
        if m == m_max:
            keep = hvecs[:, :m_min]
            gemm(B[kg:], m, keep, tmpv)
            gemm(W, m, keep, tmpw)
            for j in range(m_min):
                gs.run(tmpv[j], [(B[kg:], j)] if j else [], B[kg + j])
            W[:m_min] = tmpw[:m_min]
            H = np.diag(hvals[:m_min])
            m = m_min
            restarts += 1
        X, its, _, _, _ = engine.solve(r, [(B, kg), (u.view(1, n), 1)], delta_pcg,
                                       itmax_inner, theta=theta, negate=True)
        counter.increment(its)
        outer_solves += 1
        inner_total += its
        cx.fused(dots=[(X, None)], result=S.s[S.idx["vf"] + 2:])()
        if float(S.fetch()[0][S.idx["vf"] + 2]) == 0.0 and res > 0.0:
            # immediate indefinite direction: fall back to P M P (-r)
            qs = Slots(capacity=256)
            t0v, t1 = dev.empty(n), dev.empty(n)
            cx.project(B, kg, r, t0v, qs)
            cx.project(u.view(1, n), 1, t0v, t1, qs, name="_pu")
            cx.fused(outs=[dict(out=t1, terms=[(t1, -1.0)])])()
            t2 = dev.empty(n)
            if cx.dist:
                cx.prec_apply(prec, t1, t2)()
            else:
                prec.apply(t1, t2)
            cx.project(B, kg, t2, t0v, qs)
            cand = dev.empty(n)
            cx.project(u.view(1, n), 1, t0v, cand, qs, name="_pu")
        else:
            cand = X

    for row in locked_vecs:
        cx.gather(B[row])    # row-partitioned: every rank returns whole vectors
    order = np.argsort(locked_vals, kind="stable")
    vals = np.asarray(locked_vals)[order]
    vecs = dev.columns_to_host(B[[locked_vecs[i] for i in order]], n)
    resids = np.asarray(locked_res)[order]
    pairs = EigenPairSet(vals, vecs, resids)
    report = SolverReport(
        solver="jd", neig=neig, delta=delta, mvp=counter.count,
        outer_its=outer_solves, inner_its_total=inner_total,
        wall_seconds=time.perf_counter() - t0, converged=True,
        per_pair_residuals=resids.tolist(), eigenvalues=vals.tolist(),
        config={"delta_pcg": delta_pcg, "itmax_inner": itmax_inner, "m_min": m_min,
                "m_max": m_max, "seed": seed, "restarts": restarts,
                "mvp_outer": outer_mvps, "mvp_verify": verify_mvps},
    )
    return pairs, report
