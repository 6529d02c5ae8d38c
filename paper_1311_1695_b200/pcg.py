"""Deflated preconditioned conjugate gradients on the B200.

Mirrors the reference module pcg.py (lapeig 0.1.0):

    DeflationBasis        pcg.py:19-65   host columns (frozen) + device copy
    kernel_basis          pcg.py:68-84
    PcgOutcome            pcg.py:87-93
    pcg_solve             pcg.py:96-156  generic operator / preconditioner
                                         callables on device vectors
    jd_correction_solve   pcg.py:159-184 the JD correction equation on the
                                         DevicePcg engine

DevicePcg is the hot path: the whole PCG iteration -- projected SpMV,
projections, IC(0) apply, dots, the gamma / beta recurrences and the
indefinite / converged tests -- is a fixed sequence of device launches over
preallocated buffers.  Scalars live in a device slot file; the host reads
one status block per iteration.  A projection v - Q(Q^T v) costs no pass of
its own: Q^T v is fused into the pass that produces v and the update into
the pass that consumes it.
"""

from dataclasses import dataclass

import numpy as np

from . import _device as dev
from ._plan import Ctx, Fused, Graph, Prog, Slots

_ORTHO_TOL = 1e-10


class DeflationBasis:
    """Orthonormal columns spanning the subspace to project out."""

    __slots__ = ("columns", "_dev")

    def __init__(self, columns):
        columns = np.asarray(columns, dtype=np.float64)
        if columns.ndim != 2:
            raise ValueError("columns must be a 2-D array")
        if columns.shape[1]:
            gram = columns.T @ columns
            if np.abs(gram - np.eye(columns.shape[1])).max() > _ORTHO_TOL:
                raise ValueError("deflation columns are not orthonormal")
        self.columns = columns
        self.columns.setflags(write=False)
        self._dev = None

    @classmethod
    def empty(cls, n):
        return cls(np.zeros((n, 0)))

    @classmethod
    def single(cls, v):
        v = np.asarray(v, dtype=np.float64)
        nrm = np.linalg.norm(v)
        if nrm == 0:
            raise ValueError("cannot build a basis from the zero vector")
        return cls((v / nrm).reshape(-1, 1))

    @property
    def n(self):
        return self.columns.shape[0]

    @property
    def k(self):
        return self.columns.shape[1]

    def device(self):
        """(k, n) CUDA tensor: row j is column j (column-major n x k)."""
        if self._dev is None:
            self._dev = dev.to_device(np.ascontiguousarray(self.columns.T))
        return self._dev

    def project_out(self, v):
        """v minus its orthogonal projection onto the basis span (a fresh
        array, also when k == 0; pcg.py:55-60)."""
        on_dev = dev.is_device_array(v)
        if self.k == 0:
            return v.clone() if on_dev else np.array(v, dtype=np.float64)
        vd = dev.to_device(v)
        out = project_device(self.device(), self.k, vd)
        return out if on_dev else dev.to_host(out)

    def appended(self, u):
        """New basis with unit vector u (assumed orthogonal to the span) added."""
        u = dev.to_host(u).reshape(-1, 1)
        return DeflationBasis(np.hstack([self.columns, u]))


def project_device(q, k, v, out=None, slots=None):
    """out = v - Q (Q^T v) on the device (two fused passes)."""
    n = v.shape[0]
    S = slots or Slots(capacity=max(256, k + 8))
    name = f"_pc{k}"
    if name not in S.idx:
        S.add(name, max(k, 1))
    out = dev.empty(n) if out is None else out
    Fused(n, blocks=[(q, k, v)], result=S.s[S.idx[name]:])()
    Fused(n, outs=[dict(out=out, terms=[(v, 1.0)], upd=(q, k, S.p(name)))])()
    return out


def kernel_basis(n, labels=None):
    """Orthonormal basis of the Laplacian kernel (pcg.py:68-84)."""
    if labels is None:
        return DeflationBasis(np.full((n, 1), 1.0 / np.sqrt(n)))
    labels = np.asarray(labels, dtype=np.int64)
    if labels.shape != (n,):
        raise ValueError("labels must have one entry per node")
    ncomp = int(labels.max()) + 1
    cols = np.zeros((n, ncomp))
    sizes = np.bincount(labels, minlength=ncomp)
    cols[np.arange(n), labels] = 1.0 / np.sqrt(sizes[labels])
    return DeflationBasis(cols)


@dataclass
class PcgOutcome:
    solution: object
    iterations: int
    final_relres: float
    converged: bool
    indefinite: bool = False


# --------------------------------------------------------------- generic --
class _VecOps:
    """Small device vector helpers for the generic pcg_solve."""

    def __init__(self, n):
        self.n = n
        self.S = Slots(capacity=256)
        self.S.add("d", 8)

    def dot(self, a, b):
        Fused(self.n, dots=[(a, b)], result=self.S.s[self.S.idx["d"]:])()
        return float(self.S.fetch()[0][self.S.idx["d"]])

    def nrm(self, a):
        return float(np.sqrt(max(self.dot(a, a), 0.0)))

    def lin(self, out, terms):
        Fused(self.n, outs=[dict(out=out, terms=terms)])()
        return out


def _as_dev(y):
    return y if dev.is_device_array(y) else dev.to_device(y)


def pcg_solve(op, precond, b, tol, maxit, deflation=None, counter=None, callback=None):
    """Conjugate gradients for op(x) = b on the complement of the deflation
    basis (pcg.py:96-156).

    op(x, counter) -> y and precond (None, a callable, or an object with
    .apply) receive device tensors; numpy results are uploaded.  Iterates,
    residuals and preconditioned residuals stay projected; nonpositive
    curvature stops the iteration and flags the outcome indefinite.
    """
    host_in = not dev.is_device_array(b)
    bd = dev.to_device(b)
    n = bd.shape[0]
    V = _VecOps(n)
    if deflation is None or deflation.k == 0:
        project = lambda v: v  # noqa: E731
        bhat = bd.clone()
    else:
        project = lambda v: _as_dev(deflation.project_out(v))  # noqa: E731
        bhat = project(bd)
    if precond is None:
        psolve = lambda r: r  # noqa: E731
    elif callable(precond):
        psolve = precond
    else:
        psolve = precond.apply
    normb = V.nrm(bhat)
    if normb == 0.0:
        z = dev.zeros(n)
        return PcgOutcome(dev.to_host(z) if host_in else z, 0, 0.0, True)
    x = dev.zeros(n)
    r = bhat.clone()
    z = project(_as_dev(psolve(r)))
    rz = V.dot(r, z)
    p = z.clone()
    relres, it = 1.0, 0
    indefinite = converged = False
    while it < maxit:
        ap = project(_as_dev(op(p, counter)))
        it += 1
        pap = V.dot(p, ap)
        if pap <= 0.0:
            indefinite = True
            break
        gamma = rz / pap
        V.lin(x, [(x, 1.0), (p, gamma)])
        r = project(V.lin(dev.empty(n), [(r, 1.0), (ap, -gamma)]))
        relres = V.nrm(r) / normb
        if callback is not None:
            callback(dev.to_host(x) if host_in else x)
        if relres <= tol:
            converged = True
            break
        z = project(_as_dev(psolve(r)))
        rz_next = V.dot(r, z)
        if rz_next <= 0.0:
            indefinite = True
            break
        p = V.lin(dev.empty(n), [(z, 1.0), (p, rz_next / rz)])
        rz = rz_next
    return PcgOutcome(dev.to_host(x) if host_in else x, it, relres, converged, indefinite)


# ------------------------------------------------------------ DevicePcg --
_PCG_BATCH = 8
class DevicePcg:
    """Deflated PCG with every step on the device.

    mode "jd":    op(p) = P(A p - theta p), psolve(r) = P M P r, and the
                  PCG itself projects ap, r and z (pcg.py:159-184 + 96-156)
    mode "plain": op(p) = A p, psolve = M, PCG projects ap, r and z
                  (irlm.py:104-108)
    Q is given as up to two column blocks ((k, n) tensors, rows = columns).

    Slot groups are laid out so that every fused pass deposits its dot
    products and Q^T v coefficients exactly where the consuming pass reads
    them (result = [dots..., block dots...] is written contiguously).
    """

    def __init__(self, csr, prec, n, mode, kmax, cx=None):
        self.n, self.mode, self.kmax = n, mode, max(1, kmax)
        self.cx = cx or Ctx(n)
        self.csr = csr
        self.prec = prec
        kq = self.kmax + 1
        S = self.S = Slots(capacity=64 + 8 * (kq + 2))
        for nm in ("theta", "normb2", "normb", "pap", "rz", "rzn", "gamma", "beta",
                   "relres", "tol", "its", "zero", "t1", "t2"):
            S.add(nm)
        for nm in ("stop", "indef", "conv", "zero"):
            S.add_flag(nm)
        S.add("rr")           # "rr" is immediately followed by "cr"
        S.add("cr", kq)
        for nm in ("cb", "cz1", "cz2", "cy1", "cy2", "cr1"):
            S.add(nm, kq)
        e = dev.empty
        self.X, self.R, self.Z, self.Z0, self.P = e(n), e(n), e(n), e(n), e(n)
        self.Y, self.AP, self.T, self.Z1 = e(n), e(n), e(n), e(n)
        self._progs()
        self._sig = None
        self._hint = 4

    def _progs(self):
        S = self.S
        p = Prog(S)
        p.const("zero", 0.0)
        p.mov("normb2", "rr")
        p.sqrt("normb", "normb2")
        p.eq("t1", "normb", "zero")
        p.flag("zero", "t1")
        p.flag("stop", "t1")
        p.const("its", 0.0)
        self.p_setup = p.build()
        p = Prog(S, skip="stop")
        p.inc("its")
        p.const("zero", 0.0)
        p.le("t1", "pap", "zero")
        p.flag("indef", "t1")
        p.flagor("stop", "t1")
        p.div("gamma", "rz", "pap")
        self.p_gamma = p.build()
        p = Prog(S, skip="stop")
        p.sqrt("t1", "rr")
        p.div("relres", "t1", "normb")
        p.le("t2", "relres", "tol")
        p.flag("conv", "t2")
        p.flagor("stop", "t2")
        self.p_relres = p.build()
        p = Prog(S, skip="stop")
        p.const("zero", 0.0)
        p.le("t1", "rzn", "zero")
        p.flag("indef", "t1")
        p.flagor("stop", "t1")
        p.div("beta", "rzn", "rz")
        p.mov("rz", "rzn")
        self.p_beta = p.build()

    def _upd(self, o, coef, cscale=1.0):
        """Attach 'out -= cscale * Q c' (c at slot group `coef`)."""
        off = 0
        for i, (q, k) in enumerate(self.qb):
            o["upd" if i == 0 else "upd2"] = (q, k, self.S.p(coef, off), cscale)
            off += k
        return o

    def _qdots(self, vec):
        return [(q, k, vec) for q, k in self.qb]

    def _res(self, nm):
        return self.S.s[self.S.idx[nm]:]

    def build(self, qb):
        """(Re)build the launch plan for the projection blocks qb."""
        qb = [(q, k) for q, k in qb if k > 0]
        sig = tuple((q.data_ptr(), k) for q, k in qb)
        if sig == self._sig:
            return
        if sum(k for _, k in qb) > self.kmax + 1:
            raise ValueError("projection basis wider than the engine was built for")
        if len(qb) > 2:
            raise ValueError("at most two projection blocks")
        self._sig = sig
        self.qb = qb
        S, n, cx = self.S, self.n, self.cx
        jd = self.mode == "jd"
        has_q = bool(qb)
        stop = S.fp("stop")
        X, R, Z, Z0, P, Y, AP, T, Z1 = (self.X, self.R, self.Z, self.Z0, self.P, self.Y,
                                        self.AP, self.T, self.Z1)
        # psolve(R) -> Z  (Q^T R already in "cr")
        ps = []
        if jd and has_q:
            ps.append(cx.fused(outs=[self._upd(dict(out=T, terms=[(R, 1.0)]), "cr")],
                            skip=stop))
            ps.append(cx.prec_apply(self.prec, T, Z0, skip=stop))
        else:
            ps.append(cx.prec_apply(self.prec, R, Z0, skip=stop))
        if has_q:
            ps.append(cx.fused(blocks=self._qdots(Z0), result=self._res("cz1"), skip=stop))
            if jd:
                ps.append(cx.fused(outs=[self._upd(dict(out=Z1, terms=[(Z0, 1.0)]), "cz1")],
                                blocks=self._qdots(1), result=self._res("cz2"), skip=stop))
                zlast = lambda: self._upd(dict(out=Z, terms=[(Z1, 1.0)]), "cz2")  # noqa: E731
            else:
                zlast = lambda: self._upd(dict(out=Z, terms=[(Z0, 1.0)]), "cz1")  # noqa: E731
        else:
            zlast = lambda: dict(out=Z, terms=[(Z0, 1.0)])  # noqa: E731
        self.ps = ps
        # z of the setup also initialises P = Z and rz = R.Z
        self.zinit = cx.fused(outs=[zlast(), dict(out=P, terms=[(1, 1.0)])], dots=[(R, 1)],
                           result=self._res("rz"), skip=stop)
        body = []
        theta = S.p("theta")
        if jd:
            body.append(cx.spmv(self.csr, P, Y, theta_d=theta, skip=stop))
            if has_q:
                body.append(cx.fused(blocks=self._qdots(Y), result=self._res("cy1"), skip=stop))
                body.append(cx.fused(outs=[self._upd(dict(out=T, terms=[(Y, 1.0)]), "cy1")],
                                  blocks=self._qdots(1), result=self._res("cy2"), skip=stop))
                body.append(cx.fused(outs=[self._upd(dict(out=AP, terms=[(T, 1.0)]), "cy2")],
                                  dots=[(P, 1)], result=self._res("pap"), skip=stop,
                                  prog=self.p_gamma))
            else:
                body.append(cx.fused(outs=[dict(out=AP, terms=[(Y, 1.0)])], dots=[(P, 1)],
                                  result=self._res("pap"), skip=stop, prog=self.p_gamma))
        else:
            if len(qb) == 1:
                body.append(cx.spmv(self.csr, P, Y, q=qb[0][0], nq=qb[0][1],
                                 result=self._res("cy1"), skip=stop))
            else:
                body.append(cx.spmv(self.csr, P, Y, skip=stop))
                if has_q:
                    body.append(cx.fused(blocks=self._qdots(Y), result=self._res("cy1"),
                                      skip=stop))
            o = dict(out=AP, terms=[(Y, 1.0)])
            if has_q:
                self._upd(o, "cy1")
            body.append(cx.fused(outs=[o], dots=[(P, 1)], result=self._res("pap"), skip=stop,
                              prog=self.p_gamma))
        gam = S.p("gamma")
        if has_q:
            body.append(cx.fused(outs=[dict(out=X, terms=[(X, 1.0), (P, 1.0, gam)]),
                                       dict(out=T, terms=[(R, 1.0), (AP, -1.0, gam)])],
                              blocks=self._qdots(2), result=self._res("cr1"), skip=stop))
            # R = T - Q cr1, rr = R.R and Q^T R -> cr (rr is followed by cr)
            body.append(cx.fused(outs=[self._upd(dict(out=R, terms=[(T, 1.0)]), "cr1")],
                              dots=[(1, None)], blocks=self._qdots(1), result=self._res("rr"),
                              skip=stop, prog=self.p_relres))
        else:
            body.append(cx.fused(outs=[dict(out=X, terms=[(X, 1.0), (P, 1.0, gam)]),
                                       dict(out=R, terms=[(R, 1.0), (AP, -1.0, gam)])],
                              dots=[(2, None)], result=self._res("rr"), skip=stop,
                              prog=self.p_relres))
        body += ps
        body.append(cx.fused(outs=[zlast()], dots=[(R, 1)], result=self._res("rzn"), skip=stop,
                          prog=self.p_beta))
        body.append(cx.fused(outs=[dict(out=P, terms=[(Z, 1.0), (P, 1.0, S.p("beta"))])],
                          skip=stop))
        self.body = body
        self.body_graph = Graph(body)
        if cx.eager:
            self.body_graph.eager = True   # host-synchronous collectives in the body

    def solve(self, b, qb, tol, maxit, theta=0.0, negate=False):
        """Solve op(x) = (-b if negate else b) from x0 = 0; returns
        (X, its, relres, converged, indefinite).  X is this engine's buffer."""
        self.build(qb)
        S, cx = self.S, self.cx
        S.clear_flags()
        S.set(theta=theta, tol=tol)
        sign = -1.0 if negate else 1.0
        R, X = self.R, self.X
        if self.qb:
            cx.fused(blocks=self._qdots(b), result=self._res("cb"))()
            cx.fused(outs=[self._upd(dict(out=R, terms=[(b, sign)]), "cb", sign),
                           dict(out=X, terms=[])],
                  dots=[(1, None)], blocks=self._qdots(1), result=self._res("rr"))()
        else:
            cx.fused(outs=[dict(out=R, terms=[(b, sign)]), dict(out=X, terms=[])],
                  dots=[(1, None)], result=self._res("rr"))()
        self.p_setup()
        for f in self.ps:
            f()
        self.zinit()
        its, relres = 0, 1.0
        s, flags = S.fetch()
        if not flags[S.fidx["stop"]]:
            while its < maxit:
                # several iterations per host synchronisation: every body
                # launch skips once "stop" is set, and "its" counts only the
                # iterations that ran; the batch follows the previous solve's
                # iteration count (consecutive correction solves are alike)
                nb = max(1, min(_PCG_BATCH, maxit - its, max(2, self._hint - its)))
                for _ in range(nb):
                    self.body_graph()
                s, flags = S.fetch()
                its = int(s[S.idx["its"]])
                relres = float(s[S.idx["relres"]])
                if flags[S.fidx["stop"]]:
                    break
            self._hint = its
        if flags[S.fidx["zero"]]:
            X.zero_()
            return X, 0, 0.0, True, False
        return X, its, relres, bool(flags[S.fidx["conv"]]), bool(flags[S.fidx["indef"]])


def jd_correction_solve(a, theta, q, residual, f, tol, itmax, counter=None):
    """Approximate solve of (I - QQ')(A - theta I)(I - QQ') s = -residual
    (pcg.py:159-184); generic entry point over device vectors."""
    from .sparse import spmv
    from .ic0 import projected_precond_apply
    on_dev = dev.is_device_array(residual)
    rd = dev.to_device(residual)

    def op(x, c):
        y = spmv(a, x, c)
        V = _VecOps(x.shape[0])
        return q.project_out(V.lin(dev.empty(x.shape[0]), [(y, 1.0), (x, -float(theta))]))

    psolve = None if f is None else (lambda r: projected_precond_apply(f, q, r))
    neg = _VecOps(rd.shape[0]).lin(dev.empty(rd.shape[0]), [(rd, -1.0)])
    out = pcg_solve(op, psolve, neg, tol, itmax, deflation=q, counter=counter)
    s = out.solution
    V = _VecOps(rd.shape[0])
    if V.nrm(s) == 0.0 and V.nrm(rd) > 0.0:
        if f is not None:
            s = _as_dev(q.project_out(_as_dev(f.apply(_as_dev(q.project_out(neg))))))
        else:
            s = _as_dev(q.project_out(neg))
    return s if on_dev else dev.to_host(s)
