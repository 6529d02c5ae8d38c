"""Gram-Schmidt on the device; small dense eigenproblems on the host.

Mirrors kernels.py of the reference:

    GramSchmidtBreakdown, mgs_orthonormalize   kernels.py:18-55
    tridiag_eig, dense_sym_eig                 kernels.py:181-226

mgs_orthonormalize keeps the reference's contract (unit vector and norm;
a second sweep when the first shrank the vector below 0.7 of its length;
breakdown below 1e-14 of the input norm) but each sweep is a classical
Gram-Schmidt block projection v - Q (Q^T v) done in two fused device passes
instead of k dependent column updates -- the DGKS reorthogonalisation
criterion is designed for exactly this classical form.

The dense eigenproblems are at most m_max x m_max (JD) or ncv x ncv (IRLM)
and stay on the host (LAPACK via numpy), as SURVEY 8(a) prescribes.
"""

import numpy as np

from . import _device as dev

_REORTH_FACTOR = 0.7
_BREAKDOWN_REL = 1e-14
DENSE_EIG_MAX_DIM = 512


class GramSchmidtBreakdown(RuntimeError):
    """The candidate vector lies numerically inside the basis span."""


class DeviceGS:
    """Block classical Gram-Schmidt with DGKS reorthogonalisation on the
    device, against up to two column blocks ((k, n) tensors, rows = columns).

    Slot layout: n0 | c1[64] | n1 | c2[64] | n2 | c3[64] -- every pass
    writes its norm^2 and its Q^T v coefficients contiguously.
    """

    def __init__(self, n, slots=None, cx=None):
        from ._plan import Ctx, Slots
        self.n = n
        self.cx = cx or Ctx(n)
        self.S = slots or Slots()
        for nm in ("n0", "c1", "n1", "c2", "n2", "c3"):
            self.S.add(nm, 64 if nm[0] == "c" else 1)
        self.tmp = dev.empty(n)

    def run(self, v, blocks, out):
        """out = unit vector of v orthogonalised against blocks; returns
        (norm_out, norm_in).  blocks: list of ((k, n) tensor, k).  out may
        not alias v."""
        S, cx = self.S, self.cx
        blocks = [(q, k) for q, k in blocks if k > 0]
        ktot = sum(k for _, k in blocks)
        if ktot > 64:
            raise ValueError("Gram-Schmidt block wider than 64 columns")
        cx.fused(dots=[(v, None)], blocks=[(q, k, v) for q, k in blocks],
              result=S.s[S.idx["n0"]:])()
        nin = float(np.sqrt(S.fetch()[0][S.idx["n0"]]))
        if nin == 0.0:
            raise GramSchmidtBreakdown("zero vector cannot be orthonormalized")
        if ktot == 0:
            cx.fused(outs=[dict(out=out, terms=[(v, 1.0 / nin)])])()
            return nin, nin

        def sweep(src, dst, coef, res):
            ups, off = [], 0
            for q, k in blocks:
                ups.append((q, k, S.p(coef, off)))
                off += k
            o = dict(out=dst, terms=[(src, 1.0)], upd=ups[0])
            if len(ups) > 1:
                o["upd2"] = ups[1]
            cx.fused(outs=[o], dots=[(1, None)], blocks=[(q, k, 1) for q, k in blocks],
                  result=S.s[S.idx[res]:])()
            return float(np.sqrt(S.fetch()[0][S.idx[res]]))

        after = sweep(v, self.tmp, "c1", "n1")
        cur = self.tmp
        if after < _REORTH_FACTOR * nin:
            after = sweep(self.tmp, out, "c2", "n2")
            cur = out
        if after < _BREAKDOWN_REL * nin:
            raise GramSchmidtBreakdown(
                f"vector collapsed to {after:.3e} of its input norm {nin:.3e}")
        cx.fused(outs=[dict(out=out, terms=[(cur, 1.0 / after)])])()
        return after, nin


def mgs_orthonormalize(v, basis):
    """Orthonormalize v against the orthonormal columns of basis.

    Returns (unit vector, norm before normalization); raises
    GramSchmidtBreakdown when the remainder falls below 1e-14 of the input
    norm (kernels.py:22-55).  numpy in -> numpy out; CUDA tensors stay on
    the device (basis as an (n, k) tensor).
    """
    on_dev = dev.is_device_array(v)
    if on_dev:
        vv = v.to(dev.torch().float64).contiguous()
        b = basis
        if b.dim() == 1:
            b = b.reshape(-1, 1)
        if b.numel() and b.shape[0] != vv.shape[0]:
            raise ValueError("basis rows must match vector length")
        bt = b.t().contiguous() if b.numel() else None
        k = b.shape[1] if b.numel() else 0
    else:
        vv = np.array(v, dtype=np.float64)
        b = np.asarray(basis, dtype=np.float64)
        if b.ndim == 1:
            b = b.reshape(-1, 1)
        if b.size and b.shape[0] != vv.shape[0]:
            raise ValueError("basis rows must match vector length")
        k = b.shape[1] if b.size else 0
        bt = dev.to_device(np.ascontiguousarray(b.T)) if k else None
        vv = dev.to_device(vv)
    n = vv.shape[0]
    gs = DeviceGS(n)
    out = dev.empty(n)
    blocks = []
    for c0 in range(0, k, 64):
        blocks.append((bt[c0:c0 + 64], min(64, k - c0)))
    if len(blocks) > 2:
        raise ValueError("basis wider than 128 columns is not supported")
    nout, _ = gs.run(vv, blocks, out)
    return (out if on_dev else dev.to_host(out)), nout


def tridiag_eig(alpha, beta):
    """Eigendecomposition of a symmetric tridiagonal matrix (values
    ascending, vectors in matching columns); kernels.py:181-201."""
    alpha = np.asarray(alpha, dtype=np.float64)
    beta = np.asarray(beta, dtype=np.float64)
    m = alpha.shape[0]
    if m == 0:
        raise ValueError("empty tridiagonal")
    if beta.shape[0] != m - 1:
        raise ValueError("beta must be one entry shorter than alpha")
    t = np.diag(alpha) + np.diag(beta, 1) + np.diag(beta, -1)
    w, v = np.linalg.eigh(t)
    return w, v


def dense_sym_eig(h, max_dim=DENSE_EIG_MAX_DIM):
    """All eigenpairs of a small dense symmetric matrix, values ascending
    (kernels.py:204-226): same validation, LAPACK instead of tred2/tql2."""
    h = np.asarray(h, dtype=np.float64)
    if h.ndim != 2 or h.shape[0] != h.shape[1]:
        raise ValueError("matrix must be square")
    n = h.shape[0]
    if n == 0:
        raise ValueError("empty matrix")
    if n > max_dim:
        raise ValueError(f"dimension {n} exceeds dense solver cap {max_dim}")
    scale = max(1.0, float(np.abs(h).max()))
    if float(np.abs(h - h.T).max()) > 1e-12 * scale:
        raise ValueError("matrix is not symmetric to 1e-12 relative")
    if n == 1:
        return np.array([h[0, 0]]), np.ones((1, 1))
    w, v = np.linalg.eigh(0.5 * (h + h.T))
    return w, v
