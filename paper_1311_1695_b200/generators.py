"""Graph families of the benchmark configurations (BASELINE.json configs).

The reference package has no generators for these families
(generators.py:8-107 holds only small deterministic fixtures), so these are
new; the recipes are the ones fixed in SURVEY.md 8(d).  Every generator
returns a canonical EdgeList (i < j, sorted, unique, w > 0) that feeds both
the oracle and the device path, so the bit-exact Laplacian check is
meaningful.  All randomness comes from numpy.random.default_rng(seed), so
every graph is reproducible on any host with the same numpy.

    ba_graph            C1  Barabasi-Albert (networkx.barabasi_albert_graph)
    chung_lu_graph      C2 / C4  Chung-Lu with power-law expected degrees
    rmat_graph          C3 / C5  R-MAT (a, b, c, d) edge sampling
    config_graph(name)  the BASELINE configurations, LCC applied

plus the reference's own fixture families (generators.py:8-107: path,
cycle, complete, star, grid, and the seeded random_connected_graph /
geometric_graph that its test suite draws from), restated so the same seeds
give the same edge lists (pinned against kat_graphs.npz,
tests/test_oracle_golden.py).
"""

import numpy as np

from .graphs import EdgeList, largest_component


# ------------------------------------------------------------ small fixtures
def path_graph(n, weight=1.0):
    idx = np.arange(n - 1)
    return EdgeList(n, idx, idx + 1, np.full(n - 1, float(weight)))


def cycle_graph(n, weight=1.0):
    if n < 3:
        raise ValueError("cycle needs at least 3 nodes")
    i = np.arange(n)
    return EdgeList(n, i, (i + 1) % n, np.full(n, float(weight)))


def complete_graph(n, weight=1.0):
    i, j = np.triu_indices(n, k=1)
    return EdgeList(n, i, j, np.full(i.size, float(weight)))


def star_graph(leaves, weight=1.0):
    if leaves < 1:
        raise ValueError("star needs at least one leaf")
    j = np.arange(1, leaves + 1)
    return EdgeList(leaves + 1, np.zeros(leaves, dtype=np.int64), j, np.full(leaves, float(weight)))


def grid_graph(rows, cols, weight=1.0):
    ids = np.arange(rows * cols).reshape(rows, cols)
    i = np.concatenate([ids[:, :-1].ravel(), ids[:-1, :].ravel()])
    j = np.concatenate([ids[:, 1:].ravel(), ids[1:, :].ravel()])
    return EdgeList(rows * cols, i, j, np.full(i.size, float(weight)))


def random_connected_graph(n, extra_edges=0, seed=0, weighted=True):
    """A random tree (each node v > 0 hangs off a uniform earlier node) plus
    up to extra_edges distinct random chords, drawn with at most
    50 (extra_edges + 1) attempts; weights U(0.5, 1.5) drawn after the edges
    (reference generators.py:47-68, same default_rng call sequence)."""
    rng = np.random.default_rng(seed)
    edges = {(int(rng.integers(0, v)), v) for v in range(1, n)}
    target, tries = n - 1 + extra_edges, 0
    while len(edges) < target and tries < 50 * (extra_edges + 1):
        u, v = (int(t) for t in rng.integers(0, n, size=2))
        tries += 1
        if u != v:
            edges.add((u, v) if u < v else (v, u))
    ij = np.array(sorted(edges), dtype=np.int64).reshape(-1, 2)
    m = ij.shape[0]
    w = rng.uniform(0.5, 1.5, size=m) if weighted else np.ones(m)
    return EdgeList(n, ij[:, 0], ij[:, 1], w)


def geometric_graph(n, radius, seed=0, weighted=False):
    """Uniform points in the unit square, joined when closer than radius
    (weight 1 / (1 + distance) when weighted); while disconnected, the
    component of node 0 is joined to its nearest outside node (reference
    generators.py:71-107)."""
    from .graphs import connected_components
    rng = np.random.default_rng(seed)
    pts = rng.random((n, 2))
    d2 = ((pts[:, None, :] - pts[None, :, :]) ** 2).sum(axis=2)
    iu, ju = np.triu_indices(n, k=1)
    near = d2[iu, ju] < radius * radius
    i, j = iu[near], ju[near]
    w = 1.0 / (1.0 + np.sqrt(d2[i, j])) if weighted else np.ones(i.size)
    g = EdgeList(n, i, j, w)
    while True:
        count, labels = connected_components(g)
        if count == 1:
            return g
        inside = np.flatnonzero(labels == labels[0])
        outside = np.flatnonzero(labels != labels[0])
        k = int(np.argmin(d2[np.ix_(inside, outside)]))
        u, v = int(inside[k // outside.size]), int(outside[k % outside.size])
        wt = 1.0 / (1.0 + np.sqrt(d2[u, v])) if weighted else 1.0
        g = EdgeList(n, np.append(g.i, min(u, v)), np.append(g.j, max(u, v)),
                     np.append(g.w, wt))


# --------------------------------------------------------- canonicalisation
def _canonical(n, a, b, w=None):
    """Drop self-loops, orient (min, max), keep the first occurrence of each
    unordered pair; unit weights when w is None."""
    keep = a != b
    a, b = a[keep], b[keep]
    if w is not None:
        w = w[keep]
    lo = np.minimum(a, b).astype(np.int64)
    hi = np.maximum(a, b).astype(np.int64)
    key = lo * np.int64(n) + hi
    _, first = np.unique(key, return_index=True)   # sorted by key == (lo, hi)
    wt = np.ones(first.size) if w is None else np.asarray(w, dtype=np.float64)[first]
    return EdgeList.from_canonical(n, lo[first], hi[first], wt)


# ---------------------------------------------------------------- families
def ba_graph(n, m, seed=0):
    """Barabasi-Albert preferential attachment, unit weights (C1).

    Uses networkx.barabasi_albert_graph (the recipe the survey fixed);
    networkx ships in this image.
    """
    import networkx as nx

    g = nx.barabasi_albert_graph(n, m, seed=seed)
    e = np.array(g.edges(), dtype=np.int64).reshape(-1, 2)
    return _canonical(n, e[:, 0], e[:, 1])


def chung_lu_graph(n, gamma, mean_degree, max_degree=None, weighted=False, seed=0):
    """Chung-Lu graph with power-law expected degrees (C2, C4).

    Expected degrees w_v = (1 - u)^(-1/(gamma-1)), rescaled to the requested
    mean and capped (rescale + cap applied twice); m = round(sum w / 2)
    endpoint pairs drawn independently with probability proportional to w.
    With weighted=True the edge weights are integer counts drawn from
    Geometric(p = 0.5) after the endpoints (C4).
    """
    rng = np.random.default_rng(seed)
    u = rng.random(n)
    w = (1.0 - u) ** (-1.0 / (gamma - 1.0))
    for _ in range(2):
        w = w * (mean_degree / w.mean())
        if max_degree is not None:
            w = np.minimum(w, max_degree)
    m = int(round(w.sum() / 2.0))
    p = w / w.sum()
    a = rng.choice(n, m, p=p)
    b = rng.choice(n, m, p=p)
    wt = rng.geometric(0.5, m).astype(np.float64) if weighted else None
    return _canonical(n, a, b, wt)


def rmat_graph(scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=0):
    """R-MAT edge sampling (C3, C5), symmetrised, deduplicated, unit weights.

    For every bit position (least significant first) one uniform draw per
    edge picks the quadrant: row bit set iff r >= a + b; column bit set iff
    a <= r < a + b or r >= a + b + c.  No vertex permutation.
    """
    rng = np.random.default_rng(seed)
    n = 1 << scale
    m = edge_factor * n
    row = np.zeros(m, dtype=np.int64)
    col = np.zeros(m, dtype=np.int64)
    ab, abc = a + b, a + b + c
    for bit in range(scale):
        r = rng.random(m)
        row |= (r >= ab).astype(np.int64) << bit
        col |= (((r >= a) & (r < ab)) | (r >= abc)).astype(np.int64) << bit
    return _canonical(n, row, col)


CONFIGS = {
    "C1": dict(desc="Barabasi-Albert n=2000 m=2 seed 0, unit weights"),
    "C2": dict(desc="Chung-Lu n=22000 gamma=2.1 mean degree 4 cap 2500, LCC"),
    "C3": dict(desc="R-MAT scale 18 edge factor 8 (.57,.19,.19,.05), LCC"),
    "C4": dict(desc="weighted Chung-Lu n=1e6 gamma=2.5 mean degree 10, Geometric(0.5) weights, LCC"),
    "C5": dict(desc="R-MAT scale 26 edge factor 16, LCC"),
}


def config_graph(name, lcc=True):
    """EdgeList of a BASELINE configuration (largest component kept)."""
    if name == "C1":
        g = ba_graph(2000, 2, seed=0)
    elif name == "C2":
        g = chung_lu_graph(22000, 2.1, 4.0, max_degree=2500, seed=0)
    elif name == "C3":
        g = rmat_graph(18, 8, seed=0)
    elif name == "C4":
        g = chung_lu_graph(1_000_000, 2.5, 10.0, weighted=True, seed=0)
    elif name == "C5":
        g = rmat_graph(26, 16, seed=0)
    else:
        raise ValueError(f"unknown configuration {name!r}")
    if lcc:
        g, _ = largest_component(g)
    return g
