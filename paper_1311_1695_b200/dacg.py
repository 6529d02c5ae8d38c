"""Deflation-accelerated conjugate gradient eigensolver, on the B200.

Mirrors the reference module dacg.py (lapeig 0.1.0):

    DacgState, rq_gradient          dacg.py:21-45
    _is_parallel, _plane_minimize   dacg.py:48-96
    rq_line_search                  dacg.py:99-119
    dacg_smallest                   dacg.py:122-276  same signature, RNG
                                    stream, acceptance test, PR-beta reset,
                                    fallbacks, errors and report fields

One DACG iteration (dacg.py:171-233) is a fixed sequence of device launches
over preallocated buffers:

    IC(0) sweeps      z0 = M^{-1} g
    fused pass        C^T z0
    fused pass        z = z0 - C c;  (g - g_prev).z;  g.z
    scalar program    PR beta with reset and clamp (dacg.py:188-195)
    fused pass        p1 = -z + beta p;  C^T p1
    fused pass        p2 = p1 - C c;  x.p2
    fused pass        p = p2 - (x.p2) x;  x.x, p.p, x.p, x.Ax, p.Ax
    scalar program    parallel test (dacg.py:48-52)       -> skip flag
    SpMV              ap = A p;  p.ap, x.ap (epilogue)
    scalar program    2x2 plane pencil (dacg.py:55-96)     -> alpha, beta
    fused pass        x' = a x + b p;  ax' = a ax + b ap;  x'.x', x'.ax'
    scalar program    q' and the RQ-increase guard (dacg.py:221-225)
    fused pass        x = x'/|x'|, ax = ax'/|x'|, g = 2(ax - q x), |g|^2

and the host reads one status block (q, residual, flags) per iteration.  The
plane pencil is evaluated from the Gram dot products of {x, p, Ax, Ap}
instead of materialising the orthonormalised plane basis (the same 2x2
problem, no extra n-vector passes).  Buffers alternate between two parities
so nothing is copied.
"""

import time

import numpy as np

from . import _device as dev
from ._plan import Ctx, Fused, Graph, Prog, Slots
from ._rng import NormalStream
from .ic0 import ic0_factorize
from .pcg import kernel_basis
from .precond import device_preconditioner
from .results import EigenPairSet, SolverError, SolverReport
from .sparse import MvpCounter, device_csr, spmv

_PARALLEL_TOL = 1e-12


class DacgState:
    """Iterate, gradient and direction data for one pair's minimization."""

    __slots__ = ("x", "ax", "q", "grad", "p", "beta", "iterations")

    def __init__(self, x, ax):
        self.x = x
        self.ax = ax
        xh, axh = dev.to_host(x), dev.to_host(ax)
        self.q = float(_dots(xh, [(xh, axh)])[0])
        self.grad = 2.0 * (axh - self.q * xh)
        self.p = None
        self.beta = 0.0
        self.iterations = 0


def _dots(ref, pairs):
    """Dot products of host/device vectors computed on the device."""
    n = np.asarray(dev.to_host(ref)).shape[0]
    S = Slots(capacity=256)
    S.add("d", 8)
    tens = [(dev.to_device(a), dev.to_device(b)) for a, b in pairs]
    Fused(n, dots=tens, result=S.s[S.idx["d"]:])()
    return S.fetch()[0][S.idx["d"]:S.idx["d"] + len(pairs)].copy()


def rq_gradient(a, x, counter=None):
    """Rayleigh quotient and its gradient at x; exactly one product."""
    on_dev = dev.is_device_array(x)
    xd = dev.to_device(x)
    nrm2 = float(_dots(xd, [(xd, xd)])[0])
    if nrm2 == 0.0:
        raise ValueError("Rayleigh quotient undefined at the zero vector")
    ax = spmv(a, xd, counter)
    q = float(_dots(xd, [(xd, ax)])[0]) / nrm2
    g = dev.empty(a.n)
    Fused(a.n, outs=[dict(out=g, terms=[(ax, 2.0 / nrm2), (xd, -2.0 * q / nrm2)])])()
    return q, (g if on_dev else dev.to_host(g))


def _is_parallel(x, p):
    bxx, bpp, bxp = _dots(x, [(x, x), (p, p), (x, p)])
    return bpp == 0.0 or bxx * bpp - bxp * bxp <= _PARALLEL_TOL * bxx * bpp


def _plane_from_gram(xx, pp, xp, xax, pax, pap, xap):
    """The 2x2 plane pencil of dacg.py:55-96 from Gram dot products (host
    twin of the device scalar program)."""
    sx = np.sqrt(xx)
    pnorm = np.sqrt(pp)
    if sx == 0.0 or pnorm == 0.0:
        raise ValueError("degenerate plane: direction is parallel to the iterate")
    cproj = xp / sx
    spt = np.sqrt(max(pp - cproj * cproj, 0.0))
    if spt <= np.sqrt(_PARALLEL_TOL) * pnorm:
        raise ValueError("degenerate plane: direction is parallel to the iterate")
    a11 = xax / xx
    xapb = (xap / sx - cproj * a11) / spt
    paxb = (pax / sx - cproj * a11) / spt
    a22 = (pap - cproj * pax / sx - cproj * xap / sx + cproj * cproj * a11) / (spt * spt)
    a12 = 0.5 * (xapb + paxb)
    half = 0.5 * (a11 + a22)
    rad = float(np.hypot(0.5 * (a11 - a22), a12))
    mu = half - rad
    r1 = (a11 - mu, a12)
    r2 = (a12, a22 - mu)
    row = r1 if np.hypot(*r1) >= np.hypot(*r2) else r2
    cb, cp = row[1], -row[0]
    nrm = np.hypot(cb, cp)
    if nrm == 0.0:
        cb, cp, nrm = 1.0, 0.0, 1.0
    cb /= nrm
    cp /= nrm
    alpha = cb / sx - cp * cproj / (spt * sx)
    beta = cp / spt
    scale = np.hypot(alpha, beta)
    return float(mu), alpha / scale, beta / scale


def _plane_minimize(x, ax, p, ap):
    """Smallest Rayleigh quotient over span{x, p}: (mu, alpha, beta) with mu
    attained at alpha x + beta p.  Raises on a degenerate plane."""
    g = _dots(x, [(x, x), (p, p), (x, p), (x, ax), (p, ax), (p, ap), (x, ap)])
    return _plane_from_gram(*g)


def rq_line_search(a, x, p_dir, ax, counter=None):
    """Step t minimizing the Rayleigh quotient of x + t p_dir; one product."""
    xd, pd, axd = dev.to_device(x), dev.to_device(p_dir), dev.to_device(ax)
    pn = float(np.sqrt(_dots(pd, [(pd, pd)])[0]))
    if pn == 0.0:
        raise ValueError("degenerate plane: direction is zero")
    ps = dev.empty(a.n)
    Fused(a.n, outs=[dict(out=ps, terms=[(pd, 1.0 / pn)])])()
    ap = spmv(a, ps, counter)
    _, alpha, beta = _plane_minimize(xd, axd, ps, ap)
    if abs(alpha) <= 1e-14 * abs(beta):
        t_unit = np.copysign(1e9, beta) * (np.sign(alpha) if alpha != 0 else 1.0)
    else:
        t_unit = beta / alpha
    return float(t_unit / pn)


# ------------------------------------------------------------ device plan --
_SCALARS = ("q", "res", "gg", "num", "gz", "denom", "beta", "since", "period", "reset",
            "xx", "pp", "xp3", "xax", "pax", "pap", "xap", "xp", "mu", "al", "be", "nn", "na",
            "qn", "qold", "zero", "one", "half", "two", "tol", "sqtol", "eps14", "t0", "t1",
            "t2", "t3", "t4", "t5", "t6", "sx", "sp", "cp", "spt", "a11", "a22", "a12",
            "r1a", "r1b", "r2a", "r2b", "h1", "h2", "cb", "cpp", "nr", "xapb", "paxb",
            "iters", "xnorm2", "th", "rf2", "ran", "delta", "conv")


class _DacgPlan:
    """Prebuilt launches of one DACG iteration (two buffer parities)."""

    def __init__(self, a, f, n, kcap, comm=None):
        self.n = n
        self.cx = Ctx(n, comm)
        if self.cx.dist:
            self.csr = self.cx.comm.solver_operator(a)
            self.prec = self.cx.comm.local_preconditioner(a, f)
        else:
            self.csr = device_csr(a)
            self.prec = device_preconditioner(f, n)
        S = self.S = Slots(capacity=256 + 4 * (kcap + 2))
        for nm in _SCALARS:
            S.add(nm)
        for nm in ("stop", "par", "degen", "rqinc", "halt"):
            S.add_flag(nm)
        S.add("cz", kcap + 1)
        S.add("cpv", kcap + 1)
        S.add("cx", kcap + 1)
        e = dev.empty
        self.X = [e(n), e(n)]
        self.AX = [e(n), e(n)]
        self.G = [e(n), e(n)]
        self.Z0, self.Z, self.P, self.T, self.AP = e(n), e(n), e(n), e(n), e(n)
        self.XN, self.AXN, self.D = e(n), e(n), e(n)
        self.C = dev.zeros((kcap, n))
        self.k = 0
        self._progs()
        self.plans = {}

    def _progs(self):
        S = self.S
        # PR beta with reset and clamp (dacg.py:188-195); denom <- g.z
        p = Prog(S, skip="halt")
        p.ge("reset", "since", "period")
        p.divz("beta", "num", "denom")
        p.const("zero", 0.0)
        p.max("beta", "beta", "zero")
        p.sel("beta", "reset", "zero")
        p.sel("since", "reset", "zero")
        p.mov("denom", "gz")
        p.inc("ran")
        self.p_beta = p.build()
        # parallel test (dacg.py:48-52) -> par, stop
        p = Prog(S, skip="halt")
        p.const("zero", 0.0)
        p.const("tol", _PARALLEL_TOL)
        p.eq("t0", "pp", "zero")
        p.mul("t1", "xx", "pp")
        p.mul("t2", "xp3", "xp3")
        p.sub("t3", "t1", "t2")
        p.mul("t4", "tol", "t1")
        p.le("t5", "t3", "t4")
        p.emit("OR", p._s("t6"), p._s("t0"), p._s("t5"))
        p.flag("par", "t6")
        p.flag("stop", "t6")
        p.flagor("halt", "t6")
        self.p_par = p.build()
        # plane pencil from Gram dots (mirror of _plane_from_gram)
        p = Prog(S, skip="halt")
        p.const("zero", 0.0)
        p.const("half", 0.5)
        p.const("one", 1.0)
        p.const("sqtol", float(np.sqrt(_PARALLEL_TOL)))
        p.sqrt("sx", "xx")
        p.sqrt("sp", "pp")
        p.eq("t0", "sx", "zero")
        p.eq("t1", "sp", "zero")
        p.emit("OR", p._s("t0"), p._s("t0"), p._s("t1"))
        p.div("cp", "xp3", "sx")
        p.mul("t1", "cp", "cp")
        p.sub("t1", "pp", "t1")
        p.max("t1", "t1", "zero")
        p.sqrt("spt", "t1")
        p.mul("t2", "sqtol", "sp")
        p.le("t3", "spt", "t2")
        p.emit("OR", p._s("t0"), p._s("t0"), p._s("t3"))
        p.flag("degen", "t0")
        p.flagor("stop", "t0")
        p.flagor("halt", "t0")
        p.haltif("t0")
        p.div("a11", "xax", "xx")
        p.div("t1", "xap", "sx")
        p.mul("t2", "cp", "a11")
        p.sub("t3", "t1", "t2")
        p.div("xapb", "t3", "spt")
        p.div("t4", "pax", "sx")
        p.sub("t5", "t4", "t2")
        p.div("paxb", "t5", "spt")
        # a22 = (pap - cp*pax/sx - cp*xap/sx + cp^2 a11) / spt^2
        p.mul("t5", "cp", "t4")
        p.sub("t6", "pap", "t5")
        p.mul("t5", "cp", "t1")
        p.sub("t6", "t6", "t5")
        p.mul("t5", "cp", "t2")
        p.add("t6", "t6", "t5")
        p.mul("t5", "spt", "spt")
        p.div("a22", "t6", "t5")
        p.add("t1", "xapb", "paxb")
        p.mul("a12", "half", "t1")
        p.add("t1", "a11", "a22")
        p.mul("h1", "half", "t1")
        p.sub("t1", "a11", "a22")
        p.mul("t1", "half", "t1")
        p.hypot("t2", "t1", "a12")
        p.sub("mu", "h1", "t2")
        p.sub("r1a", "a11", "mu")
        p.mov("r1b", "a12")
        p.mov("r2a", "a12")
        p.sub("r2b", "a22", "mu")
        p.hypot("t1", "r1a", "r1b")
        p.hypot("t2", "r2a", "r2b")
        p.ge("t3", "t1", "t2")
        # row = r1 if |r1| >= |r2| else r2 ; cb = row[1], cpp = -row[0]
        p.mov("cb", "r2b")
        p.neg("cpp", "r2a")
        p.neg("t4", "r1a")
        p.sel("cb", "t3", "r1b")
        p.sel("cpp", "t3", "t4")
        p.hypot("nr", "cb", "cpp")
        p.eq("t1", "nr", "zero")
        p.sel("cb", "t1", "one")
        p.sel("cpp", "t1", "zero")
        p.sel("nr", "t1", "one")
        p.div("cb", "cb", "nr")
        p.div("cpp", "cpp", "nr")
        p.div("t1", "cb", "sx")
        p.mul("t2", "cpp", "cp")
        p.mul("t3", "spt", "sx")
        p.div("t2", "t2", "t3")
        p.sub("al", "t1", "t2")
        p.div("be", "cpp", "spt")
        p.hypot("t1", "al", "be")
        p.div("al", "al", "t1")
        p.div("be", "be", "t1")
        self.p_plane = p.build()
        # q' = x'.ax' / x'.x' and the RQ-increase guard (dacg.py:221-225)
        p = Prog(S, skip="halt")
        p.const("one", 1.0)
        p.const("eps14", 1e-14)
        p.div("qn", "na", "nn")
        p.abs("t1", "q")
        p.max("t1", "t1", "one")
        p.mul("t1", "eps14", "t1")
        p.add("t1", "q", "t1")
        p.gt("t2", "qn", "t1")
        p.flag("rqinc", "t2")
        p.flagor("stop", "t2")
        p.flagor("halt", "t2")
        p.haltif("t2")
        p.mov("qold", "q")
        p.mov("q", "qn")
        self.p_norm = p.build()
        # residual + counters; a convergence candidate (the host's test
        # res / q <= delta, same operations) halts the rest of the batch
        p = Prog(S, skip="halt")
        p.const("half", 0.5)
        p.const("zero", 0.0)
        p.sqrt("t1", "gg")
        p.mul("res", "half", "t1")
        p.inc("since")
        p.inc("iters")
        p.div("t2", "res", "q")
        p.le("t3", "t2", "delta")
        p.gt("t4", "q", "zero")
        p.emit("AND", p._s("conv"), p._s("t3"), p._s("t4"))
        p.flagor("halt", "conv")
        self.p_end = p.build()
        # batch start: clear the halt flag and the executed-iteration count
        p = Prog(S)
        p.const("zero", 0.0)
        p.flag("halt", "zero")
        p.mov("ran", "zero")
        self.p_clear = p.build()

    def plan(self, b):
        """Launch list of one iteration for parity b (x in X[b])."""
        key = (b, self.k)
        if key in self.plans:
            return self.plans[key]
        S, n, k, C = self.S, self.n, self.k, self.C
        c, o = b, 1 - b
        X, AX, G = self.X, self.AX, self.G
        Z0, Z, P, T, AP, XN, AXN, D = (self.Z0, self.Z, self.P, self.T, self.AP, self.XN,
                                       self.AXN, self.D)
        stop = S.fp("halt")   # every launch of an iteration skips once a batch halted
        res = lambda nm: S.s[S.idx[nm]:]  # noqa: E731
        L = []
        # scalar programs run in the finishing CTA of the pass whose dots
        # they consume (lg_fused_prog): no launch of their own
        cx = self.cx
        L.append(cx.prec_apply(self.prec, G[c], Z0, skip=stop))
        L.append(cx.fused(blocks=[(C, k, Z0)], result=res("cz"), skip=stop))
        # z = z0 - C cz; num = (g - g_prev).z; gz = g.z   (g_prev lives in G[o])
        L.append(cx.fused(outs=[dict(out=Z, terms=[(Z0, 1.0)], upd=(C, k, S.p("cz")))],
                       dots=[(G[c], 1, G[o]), (G[c], 1)], result=res("num"), skip=stop,
                       prog=self.p_beta))
        # p1 = -z + beta p; C^T p1
        L.append(cx.fused(outs=[dict(out=T, terms=[(Z, -1.0), (P, 1.0, S.p("beta"))])],
                       blocks=[(C, k, 1)], result=res("cpv"), skip=stop))
        # p2 = p1 - C cpv; xp = x.p2
        L.append(cx.fused(outs=[dict(out=D, terms=[(T, 1.0)], upd=(C, k, S.p("cpv")))],
                       dots=[(X[c], 1)], result=res("xp"), skip=stop))
        # p = p2 - xp x; Gram dots; parallel test
        L.append(cx.fused(outs=[dict(out=P, terms=[(D, 1.0), (X[c], -1.0, S.p("xp"))])],
                       dots=[(X[c], None), (1, None), (X[c], 1), (X[c], AX[c]), (1, AX[c])],
                       result=res("xx"), skip=stop, prog=self.p_par))
        L.append(cx.spmv(self.csr, P, AP, skip=stop))
        # pap = ap.p, xap = ap.x; plane pencil
        L.append(cx.fused(dots=[(AP, P), (AP, X[c])], result=res("pap"), skip=stop,
                       prog=self.p_plane))
        L.append(cx.fused(outs=[dict(out=XN, terms=[(X[c], 1.0, S.p("al")), (P, 1.0, S.p("be"))]),
                                dict(out=AXN, terms=[(AX[c], 1.0, S.p("al")),
                                                     (AP, 1.0, S.p("be"))])],
                       dots=[(1, None), (1, 2)], result=res("nn"), skip=stop, prog=self.p_norm))
        nn = S.p("nn")
        L.append(cx.fused(outs=[dict(out=X[o], terms=[(XN, 1.0)], post=(nn, 3)),
                                dict(out=AX[o], terms=[(AXN, 1.0)], post=(nn, 3)),
                                dict(out=G[o], terms=[(2, 2.0), (1, -2.0, S.p("q"))])],
                       dots=[(3, None)], result=res("gg"), skip=stop, prog=self.p_end))
        self.plans[key] = L
        return L

    def graph(self, b):
        """The iteration of parity b as a CUDA graph (one launch)."""
        key = ("g", b, self.k)
        g = self.plans.get(key)
        if g is None:
            g = Graph(self.plan(b))
            if self.cx.eager:
                g.eager = True   # host-synchronous collectives inside the iteration
            self.plans[key] = g
        return g


def _device_plan(a, f, n, kcap, comm=None):
    return _DacgPlan(a, f, n, kcap, comm)


def dacg_smallest(a, neig, delta=1e-6, f=None, null_basis=None,
                  maxit_per_pair=20000, *, seed=0, counter=None, x0=None, comm=None):
    """neig smallest strictly positive eigenpairs by Rayleigh quotient
    descent (dacg.py:122-276).  Each accepted iterate is verified with a
    fresh product against ||A x - q x|| / q <= delta and joined to the
    deflation set; raises with partial results attached when a pair exceeds
    maxit_per_pair.

    comm (extension, not in the reference): a dist.RowComm -- this process is
    one rank of a row-partitioned solve; f is then None or
    'fsai' (the default: FSAI as two row-partitioned products, the same
    preconditioner at every rank count), an FsaiFactor, an Ic0JacobiFactor,
    a JacobiFactor, 'jacobi' or 'block_ic0' (dist.RowComm.local_preconditioner),
    and every rank returns the same pairs."""
    with dev.solver_stream():
        return _dacg(a, neig, delta, f, null_basis, maxit_per_pair, seed, counter, x0, comm)


_BATCH = 8   # iterations launched per host synchronisation
_GRAM = 5    # plan index of the Gram-dot pass (with the parallel test)


def _dacg(a, neig, delta, f, null_basis, maxit_per_pair, seed, counter, x0, comm=None):
    t0 = time.perf_counter()
    if counter is None:
        counter = MvpCounter()
    if null_basis is None:
        null_basis = kernel_basis(a.n)
    if comm is not None and comm.world == 1 and isinstance(f, str):
        # one rank: block-Jacobi IC(0) with one block is the reference IC(0)
        from .precond import FsaiFactor, JacobiFactor
        f = {"jacobi": JacobiFactor, "fsai": FsaiFactor}.get(f, lambda _: None)(a)
    if f is None and (comm is None or comm.world == 1):
        f = ic0_factorize(a)
    if neig < 1:
        raise ValueError("neig must be at least 1")
    usable = a.n - null_basis.k
    if neig > usable:
        raise ValueError(f"asked for {neig} pairs but only {usable} exist "
                         "outside the kernel")
    rng = np.random.default_rng(seed)
    draws = NormalStream(rng, a.n)
    reset_period = max(1, a.n // 10)
    n = a.n
    kcap = null_basis.k + neig
    if kcap > 64:
        raise ValueError("more than 64 deflation columns")
    pl = _device_plan(a, f, n, kcap, comm)
    S, C, cx = pl.S, pl.C, pl.cx
    S.set(delta=delta)
    k = null_basis.k
    if k:
        C[:k] = null_basis.device()
    pl.k = k
    vals, vecs, resids, per_pair = [], [], [], []
    setup_mvps = verify_mvps = 0
    ix = S.idx
    res = lambda nm: S.s[ix[nm]:]  # noqa: E731

    for pair_idx in range(neig):
        pl.k = k
        b = 0
        X, AX, G = pl.X, pl.AX, pl.G
        if pair_idx == 0 and x0 is not None:
            start = np.asarray(dev.to_host(x0), dtype=np.float64).copy()
        else:
            start = draws.draw()
        xs = dev.to_device(start)
        # x = guard.project_out(x); x /= |x|; ax = A x; q = x.ax; g = 2(ax - q x)
        cx.project(C, k, xs, pl.D, S) if k else pl.D.copy_(xs)
        cx.fused(dots=[(pl.D, None)], result=res("xnorm2"))()
        if float(S.fetch()[0][ix["xnorm2"]]) == 0.0:
            raise SolverError(f"pair {pair_idx}: start vector lies in the deflated subspace")
        cx.fused(outs=[dict(out=X[0], terms=[(pl.D, 1.0)], post=(S.p("xnorm2"), 3))])()
        cx.spmv(pl.csr, X[0], AX[0], dots=[X[0]], result=res("q"))()
        counter.increment()
        setup_mvps += 1
        cx.fused(outs=[dict(out=G[0], terms=[(AX[0], 2.0), (X[0], -2.0, S.p("q"))]),
                       dict(out=G[1], terms=[]), dict(out=pl.P, terms=[])],
              dots=[(1, None)], result=res("gg"))()
        S.set(since=reset_period, period=reset_period, iters=0, denom=0.0)
        p_half = Prog(S)
        p_half.const("half", 0.5)
        p_half.sqrt("t1", "gg")
        p_half.mul("res", "half", "t1")
        p_half()
        iterations = 0
        accepted = None
        resv = np.inf
        q = 0.0
        s, fl = S.fetch()
        while iterations < maxit_per_pair:
            q, resv = float(s[ix["q"]]), float(s[ix["res"]])
            if q > 0 and resv / q <= delta:
                # candidate passes on cached data; confirm with a fresh product
                xc = pl.D
                if k:
                    cx.project(C, k, X[b], xc, S)
                else:
                    xc.copy_(X[b])
                cx.fused(dots=[(xc, None)], result=res("xnorm2"))()
                cx.fused(outs=[dict(out=xc, terms=[(xc, 1.0)], post=(S.p("xnorm2"), 3))])()
                w = pl.T
                cx.spmv(pl.csr, xc, w, dots=[xc], result=res("th"))()
                counter.increment()
                verify_mvps += 1
                cx.fused(outs=[dict(out=pl.AP, terms=[(w, 1.0), (xc, -1.0, S.p("th"))])],
                      dots=[(1, None)], result=res("rf2"))()
                s, _ = S.fetch()
                theta = float(s[ix["th"]])
                res_fresh = float(np.sqrt(s[ix["rf2"]]))
                if theta > 0 and res_fresh / theta <= delta:
                    accepted = (theta, None, res_fresh / theta, xc)
                    break
                # continue from the refreshed iterate (dacg.py:184-186)
                X[b].copy_(xc)
                AX[b].copy_(w)
                S.set(q=theta)
                cx.fused(outs=[dict(out=G[b], terms=[(w, 2.0), (xc, -2.0, S.p("th"))])])()
            # a batch of iterations back to back on the device: every launch
            # of an iteration skips once an earlier one halted (convergence
            # candidate, collapsed direction, degenerate plane, RQ increase),
            # so the host synchronises once per batch instead of per iteration
            nb = min(_BATCH, maxit_per_pair - iterations)
            pl.p_clear()
            for j in range(nb):
                pl.graph(b ^ (j & 1))()
            s, fl = S.fetch()
            ran = int(s[ix["ran"]])
            if ran < 1:
                raise SolverError(f"pair {pair_idx}: device batch did not run")
            counter.increment(ran - 1)
            iterations += ran - 1
            b ^= (ran - 1) & 1          # parity of the last iteration that ran
            L = pl.plan(b)
            if fl[S.fidx["par"]]:
                # collapsed direction: steepest descent, then random (dacg.py:199-212)
                retries = 0
                while True:
                    retries += 1
                    if retries == 1:
                        src, sign = pl.Z, -1.0
                    elif retries <= 3:
                        src, sign = dev.to_device(draws.draw()), 1.0
                    else:
                        raise SolverError(
                            f"pair {pair_idx}: no usable search direction at "
                            f"iteration {iterations}")
                    cx.fused(outs=[dict(out=pl.T, terms=[(src, sign)])])()
                    if k:
                        cx.project(C, k, pl.T, pl.D, S)
                    else:
                        pl.D.copy_(pl.T)
                    cx.fused(dots=[(X[b], pl.D)], result=res("xp"))()
                    pl.p_clear()
                    L[_GRAM]()   # p = p2 - (x.p2) x, Gram dots, parallel test
                    s, fl = S.fetch()
                    if not fl[S.fidx["par"]]:
                        break
                for fn in L[_GRAM + 1:]:
                    fn()
                s, fl = S.fetch()
            if fl[S.fidx["degen"]]:
                raise ValueError("degenerate plane: direction is parallel to the iterate")
            counter.increment()
            if fl[S.fidx["rqinc"]]:
                raise SolverError(
                    f"pair {pair_idx}: Rayleigh quotient increased from "
                    f"{float(s[ix['q']])!r} to {float(s[ix['qn']])!r}")
            iterations += 1
            b = 1 - b
        if accepted is None:
            for v in vecs:
                cx.gather(v)
            partial = EigenPairSet(np.asarray(vals), dev.columns_to_host(vecs, n),
                                   np.asarray(resids))
            err = SolverError(
                f"pair {pair_idx}: iteration cap {maxit_per_pair} reached "
                f"(residual {resv / q if q else np.inf:.3e}, target {delta:.1e})")
            err.partial = partial
            err.stalled_pair = pair_idx
            raise err
        theta, _, rres, xc = accepted
        vals.append(theta)
        resids.append(rres)
        per_pair.append(iterations)
        C[k].copy_(xc)
        vecs.append(C[k])   # accepted vectors stay on the device until the end
        k += 1

    for v in vecs:
        cx.gather(v)     # row-partitioned: every rank returns whole vectors
    order = np.argsort(vals, kind="stable")
    pairs = EigenPairSet(np.asarray(vals)[order], dev.columns_to_host([vecs[i] for i in order], n),
                         np.asarray(resids)[order])
    report = SolverReport(
        solver="dacg", neig=neig, delta=delta, mvp=counter.count, outer_its=0,
        inner_its_total=int(np.sum(per_pair)), wall_seconds=time.perf_counter() - t0,
        converged=True, per_pair_residuals=pairs.residuals.tolist(),
        eigenvalues=pairs.values.tolist(),
        config={"seed": seed, "maxit_per_pair": maxit_per_pair,
                "iterations_per_pair": per_pair, "mvp_setup": setup_mvps,
                "mvp_verify": verify_mvps},
    )
    return pairs, report
