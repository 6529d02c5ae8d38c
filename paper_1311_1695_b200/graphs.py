"""Weighted undirected graphs and Laplacian assembly.

Mirrors the parts of the reference graphs.py on the hot path's input side:

    EdgeList            graphs.py:28-83   canonical (i < j, lexsorted, w > 0)
    build_laplacian     graphs.py:250-263 L = D - A, explicit diagonal;
                                          assembled on the device
                                          (lg_build_laplacian), bit-exact
    connected_components / largest_component
                        graphs.py:278-316 same numbering (components by
                                          smallest node, ties -> smallest id)

File loaders, stats and Matrix Market output (graphs.py:86-247,319-361) are
one-time host ingest and stay out of scope.
"""

import numpy as np

from . import _native as nat
from . import _device as dev
from .sparse import CsrMatrix


class EdgeList:
    """Canonical weighted edge list on nodes 0..n_nodes-1 (graphs.py:28-83)."""

    __slots__ = ("n_nodes", "i", "j", "w")

    def __init__(self, n_nodes, i, j, w):
        n_nodes = int(n_nodes)
        i = np.array(i, dtype=np.int64)
        j = np.array(j, dtype=np.int64)
        w = np.array(w, dtype=np.float64)
        if n_nodes < 1:
            raise ValueError("graph needs at least one node")
        if not (i.shape == j.shape == w.shape) or i.ndim != 1:
            raise ValueError("i, j, w must be 1-D arrays of equal length")
        if i.size:
            lo_bad = min(i.min(), j.min()) < 0
            hi_bad = max(i.max(), j.max()) >= n_nodes
            if lo_bad or hi_bad:
                raise ValueError("node index out of range")
            loops = np.flatnonzero(i == j)
            if loops.size:
                raise ValueError(f"self-loop at node {i[loops[0]]}")
            bad = np.flatnonzero(w <= 0)
            if bad.size:
                k = int(bad[0])
                raise ValueError(f"nonpositive weight {w[k]} on edge ({i[k]}, {j[k]})")
            lo = np.minimum(i, j)
            hi = np.maximum(i, j)
            order = np.lexsort((hi, lo))
            i, j, w = lo[order], hi[order], w[order]
            dup = np.flatnonzero((i[1:] == i[:-1]) & (j[1:] == j[:-1]))
            if dup.size:
                k = int(dup[0])
                raise ValueError(f"duplicate edge ({i[k]}, {j[k]})")
        self.n_nodes = n_nodes
        self.i, self.j, self.w = i, j, w
        for arr in (self.i, self.j, self.w):
            arr.setflags(write=False)

    @classmethod
    def from_pairs(cls, n_nodes, triples):
        triples = list(triples)
        if not triples:
            return cls(n_nodes, [], [], [])
        i, j, w = zip(*triples)
        return cls(n_nodes, i, j, w)

    @classmethod
    def from_canonical(cls, n_nodes, i, j, w):
        """Wrap arrays already in canonical form (checked cheaply)."""
        g = cls.__new__(cls)
        g.n_nodes = int(n_nodes)
        g.i = np.ascontiguousarray(i, dtype=np.int64)
        g.j = np.ascontiguousarray(j, dtype=np.int64)
        g.w = np.ascontiguousarray(w, dtype=np.float64)
        if g.i.size:
            if not (np.all(g.i < g.j) and g.i.min() >= 0 and g.j.max() < g.n_nodes
                    and np.all(g.w > 0)):
                raise ValueError("edges are not canonical")
            key = g.i * g.n_nodes + g.j
            if np.any(key[1:] <= key[:-1]):
                raise ValueError("edges are not sorted / unique")
        for arr in (g.i, g.j, g.w):
            arr.setflags(write=False)
        return g

    @property
    def m(self):
        return int(self.i.size)

    def pairs(self):
        return list(zip(self.i.tolist(), self.j.tolist(), self.w.tolist()))


def build_laplacian(g):
    """Weighted Laplacian L = D - A as a symmetric CsrMatrix.

    Assembled on the device; every diagonal entry is stored (nnz = n + 2m)
    and degrees are summed in the reference's order, so the arrays equal
    graphs.build_laplacian's bit for bit.
    """
    dev.require_cuda()
    n, m = g.n_nodes, g.m
    nnz = n + 2 * m
    rp = np.empty(n + 1, dtype=np.int64)
    col = np.empty(nnz, dtype=np.int64)
    val = np.empty(nnz, dtype=np.float64)
    gi = np.ascontiguousarray(g.i, dtype=np.int64)
    gj = np.ascontiguousarray(g.j, dtype=np.int64)
    gw = np.ascontiguousarray(g.w, dtype=np.float64)
    nat.call("lg_build_laplacian", n, m, gi.ctypes.data if m else None,
             gj.ctypes.data if m else None, gw.ctypes.data if m else None,
             rp.ctypes.data, col.ctypes.data, val.ctypes.data)
    return CsrMatrix(n, rp, col, val, symmetric=True)


def connected_components(g):
    """(count, labels); components numbered by their smallest node."""
    from scipy.sparse import coo_matrix
    from scipy.sparse.csgraph import connected_components as cc

    n = g.n_nodes
    adj = coo_matrix((np.ones(g.m), (g.i, g.j)), shape=(n, n)).tocsr()
    count, lab = cc(adj, directed=False)
    # renumber by smallest member node
    first = np.full(count, n, dtype=np.int64)
    np.minimum.at(first, lab, np.arange(n))
    order = np.argsort(first, kind="stable")
    remap = np.empty(count, dtype=np.int64)
    remap[order] = np.arange(count)
    return int(count), remap[lab]


def largest_component(g):
    """Restrict g to its largest component (ties: smallest component id)."""
    count, labels = connected_components(g)
    sizes = np.bincount(labels, minlength=count)
    keep_label = int(np.argmax(sizes))
    keep = labels == keep_label
    node_map = np.full(g.n_nodes, -1, dtype=np.int64)
    node_map[keep] = np.arange(int(keep.sum()))
    mask = keep[g.i]
    sub = EdgeList.from_canonical(int(keep.sum()), node_map[g.i[mask]], node_map[g.j[mask]],
                                  g.w[mask])
    return sub, node_map
