"""Weighted undirected graphs and Laplacian assembly.

Mirrors the parts of the reference graphs.py on the hot path's input side:

    EdgeList            graphs.py:28-83   canonical (i < j, lexsorted, w > 0)
    build_laplacian     graphs.py:250-263 L = D - A, explicit diagonal;
                                          assembled on the device
                                          (lg_build_laplacian), bit-exact
    connected_components / largest_component
                        graphs.py:278-316 same numbering (components by
                                          smallest node, ties -> smallest id)

    GraphFormatError, load_edge_list
                        graphs.py:18-25,126-247 text edge lists and Matrix
                                          Market files parsed in C++
                                          (lg_graph_parse, lg_load.cu): same
                                          rules, messages and line numbers
    GraphStats, stats, csr_connected_components, write_matrix_market
                        graphs.py:86-92,319-361
"""

import ctypes
import io
from dataclasses import dataclass
from pathlib import Path

import numpy as np

from . import _native as nat
from . import _device as dev
from .sparse import CsrMatrix


class GraphFormatError(ValueError):
    """Malformed graph input; carries a 1-based line number when known
    (graphs.py:18-25)."""

    def __init__(self, message, line=None):
        self.line = line
        if line is not None:
            message = f"line {line}: {message}"
        super().__init__(message)


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


@dataclass(frozen=True)
class GraphStats:
    n: int
    nnz: int
    anzr: float
    components: int


def load_edge_list(source, format="edgelist", symmetrize=False):
    """Read a graph from a path or open text stream (graphs.py:231-247).

    format is "edgelist" (first line n, then 'i j w' lines, # comments) or
    "mtx" (Matrix Market coordinate; diagonal entries are dropped,
    off-diagonal magnitudes become weights).  The text is parsed by the
    library's C++ parser (lg_graph_parse); errors raise GraphFormatError with
    the reference's message and 1-based line number.
    """
    if format not in ("edgelist", "mtx"):
        raise ValueError(f"unknown format {format!r}")
    if isinstance(source, (str, Path)):
        with open(source, "rb") as fh:
            data = fh.read()
        data.decode("utf-8")          # same encoding errors as the reference
    elif isinstance(source, bytes):
        data = source
        data.decode("utf-8")
    else:
        text = source.read()
        data = text.encode("utf-8") if isinstance(text, str) else bytes(text)
    # universal newlines, as Python's text I/O reads files
    if b"\r" in data:
        data = data.replace(b"\r\n", b"\n").replace(b"\r", b"\n")
    lib = nat.load()
    n, m = ctypes.c_int64(), ctypes.c_int64()
    pi, pj, pw = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_void_p()
    line = ctypes.c_int64()
    rc = lib.lg_graph_parse(data, len(data), 0 if format == "edgelist" else 1,
                            1 if symmetrize else 0, ctypes.byref(n), ctypes.byref(m),
                            ctypes.byref(pi), ctypes.byref(pj), ctypes.byref(pw),
                            ctypes.byref(line))
    if rc == nat.LG_EFORMAT:
        raise GraphFormatError(nat.last_error(), line.value or None)
    nat.check(rc, "lg_graph_parse")
    try:
        mm = m.value
        i = np.ctypeslib.as_array(ctypes.cast(pi, ctypes.POINTER(ctypes.c_int64)),
                                  (max(mm, 1),))[:mm].copy()
        j = np.ctypeslib.as_array(ctypes.cast(pj, ctypes.POINTER(ctypes.c_int64)),
                                  (max(mm, 1),))[:mm].copy()
        w = np.ctypeslib.as_array(ctypes.cast(pw, ctypes.POINTER(ctypes.c_double)),
                                  (max(mm, 1),))[:mm].copy()
    finally:
        for p in (pi, pj, pw):
            lib.lg_host_free(p)
    return EdgeList.from_canonical(n.value, i, j, w)


def stats(g):
    """Size summary: n, Laplacian nonzeros n + 2m, average per row,
    components (graphs.py:319-323)."""
    count, _ = connected_components(g)
    nnz = g.n_nodes + 2 * g.m
    return GraphStats(n=g.n_nodes, nnz=nnz, anzr=nnz / g.n_nodes, components=count)


def csr_connected_components(a):
    """Component count and labels from the off-diagonal pattern of a CSR
    matrix (graphs.py:326-344); components numbered by their smallest node."""
    rp = np.asarray(a.row_ptr)
    col = np.asarray(a.col_idx)
    n = int(a.n)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    off = rows != col
    lo = np.minimum(rows[off], col[off])
    hi = np.maximum(rows[off], col[off])
    key = np.unique(lo * max(n, 1) + hi)
    g = EdgeList.from_canonical(n, key // max(n, 1), key % max(n, 1), np.ones(key.size))
    return connected_components(g)


def write_matrix_market(a, stream=None):
    """Serialize a symmetric CSR matrix in coordinate format, lower triangle
    (graphs.py:347-361); returns the text when no stream is given."""
    rp = np.asarray(a.row_ptr)
    col = np.asarray(a.col_idx)
    val = np.asarray(a.values, dtype=np.float64)
    n = int(a.n)
    rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(rp))
    keep = col <= rows
    out = io.StringIO() if stream is None else stream
    out.write("%%MatrixMarket matrix coordinate real symmetric\n")
    out.write(f"{n} {n} {int(keep.sum())}\n")
    out.writelines(f"{i + 1} {j + 1} {float(v)!r}\n"
                   for i, j, v in zip(rows[keep].tolist(), col[keep].tolist(),
                                      val[keep].tolist()))
    return out.getvalue() if stream is None else None
