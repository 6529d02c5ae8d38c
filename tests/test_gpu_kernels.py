"""Device kernels vs the CPU oracle (parity tests proper, through the C ABI).

Tolerances: Laplacian assembly and the IC(0) factor are bit-exact; SpMV and
the IC(0) apply differ from the reference only in summation order, so they
are held to 1e-13 (SpMV) / 1e-12 (apply) relative to the largest entry;
reductions are deterministic (bitwise equal run to run).
"""

import hashlib
import os
from pathlib import Path

import numpy as np
import pytest

from oracle import lapeig_oracle as O
from tests.conftest import golden_config, kat_edges

ROOT = Path(__file__).resolve().parent.parent

pytestmark = pytest.mark.gpu

KAT = ["P3", "P4", "P10w", "C4", "C7", "K3", "K6", "S4", "S9", "grid4x5", "rand15",
       "rand50", "rand200", "geo1000"]


def sha(*arrays):
    h = hashlib.sha256()
    for a in arrays:
        h.update(np.ascontiguousarray(a).tobytes())
    return h.hexdigest()


@pytest.fixture(scope="module")
def L():
    import paper_1311_1695_b200 as lib
    return lib


def edge_list(L, graphs, name):
    n, i, j, w = kat_edges(graphs, name)
    return L.graphs.EdgeList.from_canonical(n, i, j, w)


@pytest.mark.parametrize("name", KAT)
def test_build_laplacian_bit_exact(L, kat, name):
    graphs, arrays, _ = kat
    a = L.build_laplacian(edge_list(L, graphs, name))
    assert np.array_equal(a.row_ptr, arrays[name + "_rp"])
    assert np.array_equal(a.col_idx, arrays[name + "_col"])
    assert np.array_equal(a.values.view(np.int64), arrays[name + "_val"].view(np.int64))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_build_laplacian_configs_bit_exact(L, cfg):
    ref = golden_config(cfg)
    g = L.config_graph(cfg)
    a = L.build_laplacian(g)
    assert sha(a.row_ptr, a.col_idx, a.values) == ref["csr_sha256"]
    assert sha(a.diagonal()) == ref["degree_sha256"]
    d = a.device()
    rp, ci, va = d.download()
    assert np.array_equal(rp, a.row_ptr) and np.array_equal(ci, a.col_idx)
    assert np.array_equal(va.view(np.int64), a.values.view(np.int64))


@pytest.mark.parametrize("name", KAT)
def test_spmv_matches_oracle(L, kat, name):
    graphs, arrays, _ = kat
    a = L.build_laplacian(edge_list(L, graphs, name))
    x = arrays[name + "_x"]
    y = L.spmv(a, x)
    want = arrays[name + "_spmv"]
    assert np.max(np.abs(y - want)) <= 1e-13 * max(1.0, np.max(np.abs(want)))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_spmv_configs(L, cfg):
    ref = golden_config(cfg)
    g = L.config_graph(cfg)
    a = L.build_laplacian(g)
    x = np.random.default_rng(0).standard_normal(a.n)
    y = L.spmv(a, x)
    oa = O.Csr(a.n, a.row_ptr, a.col_idx, a.values)
    want = O.spmv(oa, x)
    assert np.max(np.abs(y - want)) <= 1e-13 * np.max(np.abs(want))
    # size-independent properties: L e = 0 (rows sum to zero), linearity
    e = np.ones(a.n)
    assert np.max(np.abs(L.spmv(a, e))) <= 1e-12 * np.max(np.abs(a.values))
    x2 = np.random.default_rng(1).standard_normal(a.n)
    y12 = L.spmv(a, 2.0 * x - 3.0 * x2)
    assert np.max(np.abs(y12 - (2.0 * y - 3.0 * L.spmv(a, x2)))) <= 1e-12 * np.max(np.abs(y12))
    assert abs(float(y.sum()) - ref["spmv_x_seed0"]["sum"]) <= 1e-9 * ref["spmv_x_seed0"]["norm"]


def test_spmv_deterministic_and_counted(L, kat):
    graphs, _, _ = kat
    import torch
    a = L.build_laplacian(L.config_graph("C2"))
    x = torch.randn(a.n, dtype=torch.float64, device="cuda")
    c = L.MvpCounter()
    y1 = L.spmv(a, x, c)
    y2 = L.spmv(a, x, c)
    assert c.count == 2 and torch.equal(y1, y2) and y1.is_cuda
    with pytest.raises(ValueError):
        L.spmv(a, np.ones(a.n + 1), c)
    assert c.count == 2


def test_spmv_general_csr_edge_cases(L):
    # empty rows, a single long row (long-row split path), non-symmetric
    n = 5000
    rng = np.random.default_rng(3)
    rows = np.concatenate([np.zeros(4500, dtype=np.int64), rng.integers(0, n, 3000)])
    cols = np.concatenate([np.arange(4500), rng.integers(0, n, 3000)])
    key = np.unique(rows * n + cols)
    rows, cols = key // n, key % n
    vals = rng.standard_normal(rows.size)
    a = L.CsrMatrix.from_coo(n, rows, cols, vals)
    x = rng.standard_normal(n)
    want = O.spmv(O.Csr(n, a.row_ptr, a.col_idx, a.values), x)
    y = L.spmv(a, x)
    assert np.max(np.abs(y - want)) <= 1e-13 * np.max(np.abs(want))
    assert L.spmv(L.CsrMatrix(0, [0], [], []), np.zeros(0)).shape == (0,)
    one = L.CsrMatrix(1, [0, 1], [0], [2.5])
    assert L.spmv(one, np.array([2.0]))[0] == 5.0


def test_spmv_theta_and_epilogue_dots(L):
    import torch
    from paper_1311_1695_b200._plan import Slots, Spmv
    from paper_1311_1695_b200 import _device as dev
    a = L.build_laplacian(L.config_graph("C4"))   # has long rows
    d = a.device()
    assert d.nlong > 0
    n = a.n
    x = torch.randn(n, dtype=torch.float64, device="cuda")
    u = torch.randn(n, dtype=torch.float64, device="cuda")
    Q = torch.randn(3, n, dtype=torch.float64, device="cuda")
    S = Slots()
    S.add("th")
    S.add("out", 8)
    S.set(th=0.75)
    y = dev.empty(n)
    Spmv(d, x, y, theta=0.25, theta_d=S.p("th"), dots=[u, None], q=Q, nq=3,
         result=S.s[S.idx["out"]:])()
    s = S.fetch()[0][S.idx["out"]:S.idx["out"] + 5].copy()
    yh = O.spmv(O.Csr(n, a.row_ptr, a.col_idx, a.values), x.cpu().numpy()) - 1.0 * x.cpu().numpy()
    assert np.max(np.abs(y.cpu().numpy() - yh)) <= 1e-12 * np.max(np.abs(yh))
    want = np.concatenate([[yh @ u.cpu().numpy(), yh @ yh], Q.cpu().numpy() @ yh])
    assert np.max(np.abs(s - want) / np.abs(want)) <= 1e-12
    # bitwise deterministic epilogue
    Spmv(d, x, y, theta=0.25, theta_d=S.p("th"), dots=[u, None], q=Q, nq=3,
         result=S.s[S.idx["out"]:])()
    assert np.array_equal(S.fetch()[0][S.idx["out"]:S.idx["out"] + 5], s)


def test_fused_pass_terms_updates_dots(L):
    import torch
    from paper_1311_1695_b200._plan import Fused, Slots
    from paper_1311_1695_b200 import _device as dev
    n = 300_001
    g = torch.Generator(device="cuda").manual_seed(0)
    v = [torch.randn(n, dtype=torch.float64, device="cuda", generator=g) for _ in range(4)]
    Q1 = torch.randn(5, n, dtype=torch.float64, device="cuda", generator=g)
    Q2 = torch.randn(2, n, dtype=torch.float64, device="cuda", generator=g)
    S = Slots()
    S.add("a", 2)
    S.add("c1", 5)
    S.add("c2", 2)
    S.add("r", 40)
    S.set(a=1.5)
    S.set_vec("c1", [0.1, -0.2, 0.3, 0.4, -0.5])
    S.set_vec("c2", [2.0, -1.0])
    S.s[S.idx["a"] + 1] = 4.0
    o0, o1, o2 = dev.empty(n), dev.empty(n), dev.empty(n)
    Fused(n, outs=[dict(out=o0, terms=[(v[0], 2.0), (v[1], -1.0, S.p("a"))],
                        upd=(Q1, 5, S.p("c1"), 0.5), upd2=(Q2, 2, S.p("c2"))),
                   dict(out=o1, terms=[(1, 1.0), (v[2], 3.0)], post=(S.p("a", 1), 3)),
                   dict(out=o2, terms=[(2, 1.0), (1, -1.0)], post=(S.p("a"), 2))],
          dots=[(1, None), (v[3], 2, v[0]), (3, v[1])],
          blocks=[(Q1, 5, 1), (Q2, 2, v[3])], result=S.s[S.idx["r"]:])()
    h = lambda t: t.cpu().numpy()  # noqa: E731
    V = [h(t) for t in v]
    q1, q2 = h(Q1), h(Q2)
    w0 = 2 * V[0] - 1.5 * V[1] - 0.5 * (q1.T @ np.array([0.1, -0.2, 0.3, 0.4, -0.5])) \
        - 0.5 * (q2.T @ np.array([2.0, -1.0]))
    w1 = (w0 + 3 * V[2]) / 2.0
    w2 = (w1 - w0) / 1.5
    for got, want in ((o0, w0), (o1, w1), (o2, w2)):
        assert np.max(np.abs(h(got) - want)) <= 1e-13 * np.max(np.abs(want))
    res = S.fetch()[0][S.idx["r"]:S.idx["r"] + 10]
    want = np.concatenate([[w0 @ w0, (V[3] - V[0]) @ w1, w2 @ V[1]], q1 @ w0, q2 @ V[3]])
    assert np.max(np.abs(res - want) / np.maximum(1.0, np.abs(want))) <= 1e-11


def test_fused_skip_predicate(L):
    import torch
    from paper_1311_1695_b200._plan import Fused, Slots
    n = 1000
    S = Slots(flags=["stop"])
    x = torch.ones(n, dtype=torch.float64, device="cuda")
    y = torch.zeros(n, dtype=torch.float64, device="cuda")
    f = Fused(n, outs=[dict(out=y, terms=[(x, 2.0)])], skip=S.fp("stop"))
    S.setflag("stop", 1)
    f()
    assert float(y.sum()) == 0.0
    S.setflag("stop", 0)
    f()
    assert float(y.sum()) == 2.0 * n


def test_scalar_interpreter(L):
    from paper_1311_1695_b200._plan import Prog, Slots
    S = Slots(flags=["f"])
    p = Prog(S)
    p.const("a", 3.0)
    p.const("b", 4.0)
    p.hypot("h", "a", "b")
    p.sqrt("s", "b")
    p.divz("dz", "a", "zero")
    p.le("le", "a", "b")
    p.flag("f", "le")
    p.sel("a", "le", "b")
    p.max("m", "h", "b")
    p.haltif("le")
    p.const("never", 1.0)
    p()
    h, s, dz, a, m, never = S.read("h", "s", "dz", "a", "m", "never")
    assert (h, s, dz, a, m, never) == (5.0, 2.0, 0.0, 4.0, 5.0, 0.0)
    assert S.fetch()[1][S.fidx["f"]] == 1


@pytest.mark.parametrize("name", KAT)
def test_ic0_apply_matches_oracle(L, kat, name):
    graphs, arrays, _ = kat
    a = L.build_laplacian(edge_list(L, graphs, name))
    f = L.ic0_factorize(a)
    assert np.array_equal(f.l.values.view(np.int64), arrays[name + "_lval"].view(np.int64))
    z = f.apply(arrays[name + "_x"])
    want = arrays[name + "_ic0"]
    assert np.max(np.abs(z - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3", "C4"])
def test_ic0_configs(L, cfg):
    import torch
    ref = golden_config(cfg)
    a = L.build_laplacian(L.config_graph(cfg))
    f = L.ic0_factorize(a)
    assert sha(f.l.row_ptr, f.l.col_idx, f.l.values) == ref["ic0_sha256"]
    x = np.random.default_rng(0).standard_normal(a.n)
    z = f.apply(x)
    assert abs(np.linalg.norm(z) - ref["ic0_apply_x_seed0"]["norm"]) <= \
        1e-12 * ref["ic0_apply_x_seed0"]["norm"]
    assert np.allclose(z[:8], ref["ic0_apply_x_seed0"]["head"], rtol=1e-11, atol=0)
    # elementwise against the oracle's SuperLU apply of the same factor
    # (ic0.py:40-45 restated), relative to the largest entry
    zr = O.Ic0(a.n, f.l.row_ptr, f.l.col_idx, f.l.values).apply(x)
    assert np.max(np.abs(z - zr)) <= 1e-12 * np.max(np.abs(zr))
    # L L^T z = x (inverse property, size independent)
    Lm = O.Csr(a.n, f.l.row_ptr, f.l.col_idx, f.l.values)
    import scipy.sparse as sp
    M = sp.csr_matrix((f.l.values, f.l.col_idx, f.l.row_ptr), shape=(a.n, a.n))
    back = M @ (M.T @ z)
    assert np.max(np.abs(back - x)) <= 1e-10 * np.max(np.abs(x))
    # deterministic and z may alias r on the device
    xd = torch.from_numpy(x).cuda()
    z1 = f.apply(xd)
    z2 = f.apply(xd)
    assert torch.equal(z1, z2)
    d = f.device()
    d.apply(xd, xd)
    assert torch.equal(xd, z1)
    del Lm


@pytest.mark.parametrize("mc", [False, True])
def test_ic0_dataflow_state_handoff(L, mc):
    """The dataflow sweeps re-arm each other's scratch state (x sentinels,
    counters, hub slots): repeated applies, skipped applies, in-place applies
    and an interleaved level-barrier apply (the trace path) must all give the
    same bits."""
    import ctypes
    import torch
    from paper_1311_1695_b200 import _device as dev, _native as nat
    a = L.build_laplacian(L.config_graph("C2"))
    f = L.ic0_factorize_multicolor(a) if mc else L.ic0_factorize(a)
    d = f.device()
    d.set_mode(0)                                   # whatever LG_SWEEP_CTA says
    rng = np.random.default_rng(3)
    xs = [torch.from_numpy(rng.standard_normal(a.n)).cuda() for _ in range(3)]
    want = [f.apply(x.cpu().numpy()) for x in xs]
    ref = [d.apply(x, dev.empty(a.n)).clone() for x in xs]
    for w, r in zip(want, ref):
        assert np.max(np.abs(r.cpu().numpy() - w)) <= 1e-12 * np.max(np.abs(w))
    skip = torch.ones(1, dtype=torch.int32, device="cuda")
    z = torch.full((a.n,), 7.0, dtype=torch.float64, device="cuda")
    d.apply_raw(xs[0].data_ptr(), z.data_ptr(), skip.data_ptr(), dev.stream_ptr())
    assert torch.all(z == 7.0)                      # skipped: untouched
    assert torch.equal(d.apply(xs[1], dev.empty(a.n)), ref[1])
    lib = nat.load()
    lib.lg_ic0_trace(d.handle, 1, None, 0)          # level-barrier path
    assert torch.equal(d.apply(xs[2], dev.empty(a.n)), ref[2])
    lib.lg_ic0_trace(d.handle, 0, None, 0)          # back to the dataflow path
    assert torch.equal(d.apply(xs[0], dev.empty(a.n)), ref[0])
    y = xs[1].clone()
    d.apply(y, y)                                   # z aliases r
    assert torch.equal(y, ref[1])
    assert torch.equal(d.apply(xs[2], dev.empty(a.n)), ref[2])


@pytest.mark.parametrize("cfg,mc", [("C1", False), ("C2", False), ("C2", True), ("C3", False)])
def test_ic0_resident_sweep_same_bits(L, cfg, mc):
    """The resident one-CTA sweep (both triangles in one launch, levels
    separated by CTA barriers) walks the dataflow sweep's tasks in the same
    summation order: bitwise the same z, whichever ran before, with skipped
    and in-place applies, and against the oracle's apply (ic0.py:40-45)."""
    import torch
    from paper_1311_1695_b200 import _device as dev
    a = L.build_laplacian(L.config_graph(cfg))
    f = L.ic0_factorize_multicolor(a) if mc else L.ic0_factorize(a)
    d = f.device()
    rng = np.random.default_rng(5)
    xs = [torch.from_numpy(rng.standard_normal(a.n)).cuda() for _ in range(3)]
    d.set_mode(0)
    flow = [d.apply(x, dev.empty(a.n)).clone() for x in xs]
    assert d.set_mode(1) == 0
    for x, w in zip(xs, flow):
        assert torch.equal(d.apply(x, dev.empty(a.n)), w)
    d.set_mode(0)                                   # back: the dataflow state is re-armed
    assert torch.equal(d.apply(xs[1], dev.empty(a.n)), flow[1])
    d.set_mode(1)
    skip = torch.ones(1, dtype=torch.int32, device="cuda")
    z = torch.full((a.n,), 7.0, dtype=torch.float64, device="cuda")
    d.apply_raw(xs[0].data_ptr(), z.data_ptr(), skip.data_ptr(), dev.stream_ptr())
    assert torch.all(z == 7.0)
    y = xs[2].clone()
    d.apply(y, y)                                   # z aliases r
    assert torch.equal(y, flow[2])
    for nthreads in (1, 2):                          # repeated applies
        assert torch.equal(d.apply(xs[0], dev.empty(a.n)), flow[0])
    if not mc:
        zr = O.Ic0(a.n, f.l.row_ptr, f.l.col_idx, f.l.values).apply(xs[0].cpu().numpy())
        assert np.max(np.abs(flow[0].cpu().numpy() - zr)) <= 1e-12 * np.max(np.abs(zr))


@pytest.mark.parametrize("name", KAT)
def test_ic0_resident_sweep_fixtures(L, kat, name):
    """Same on the reference's fixture graphs (stars and hubs included):
    resident and dataflow sweeps agree bit for bit and match the golden apply."""
    graphs, arrays, _ = kat
    a = L.build_laplacian(edge_list(L, graphs, name))
    f = L.ic0_factorize(a)
    d = f.device()
    import torch
    x = torch.from_numpy(np.ascontiguousarray(arrays[name + "_x"])).cuda()
    d.set_mode(0)
    z0 = d.apply(x).clone()
    d.set_mode(1)
    z1 = d.apply(x).clone()
    assert torch.equal(z0, z1)
    want = arrays[name + "_ic0"]
    assert np.max(np.abs(z1.cpu().numpy() - want)) <= 1e-12 * np.max(np.abs(want))


@pytest.mark.parametrize("cfg", ["C1", "C2", "C3"])
def test_ic0_level_merging(L, cfg, monkeypatch):
    """The device applies a level-merged form of the factor (odd-level rows
    split off a partial sum of their early inputs, even-level rows substitute
    the level below): shallower sweeps, the same z to roundoff -- against the
    factor's own sweeps (LG_IC0_MERGE=0), against the oracle (ic0.py:40-45),
    for every pass count, in place, and for a permuted (multicolour) factor."""
    import torch
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.ic0 import DeviceIc0
    a = L.build_laplacian(L.config_graph(cfg))
    f = L.ic0_factorize(a)
    x = np.random.default_rng(11).standard_normal(a.n)
    xd = torch.from_numpy(x).cuda()
    zr = O.Ic0(a.n, f.l.row_ptr, f.l.col_idx, f.l.values).apply(x)
    scale = np.max(np.abs(zr))
    monkeypatch.setenv("LG_IC0_MERGE", "0")
    d0 = DeviceIc0(f.l)
    assert d0.sweep_levels == (d0.levels, d0.levels) and d0.sweep_entries == 2 * (d0.nnz_l - a.n)
    z0 = d0.apply(xd).cpu().numpy()
    assert np.max(np.abs(z0 - zr)) <= 1e-12 * scale
    prev = d0.sweep_levels
    for passes in (1, 2, 3):
        monkeypatch.setenv("LG_IC0_MERGE", str(passes))
        d = DeviceIc0(f.l)
        assert d.levels == d0.levels                      # the factor's own depth is reported unchanged
        assert max(d.sweep_levels) < max(prev) and d.sweep_entries > d0.sweep_entries
        prev = d.sweep_levels
        z = d.apply(xd)
        assert np.max(np.abs(z.cpu().numpy() - zr)) <= 1e-12 * scale
        assert np.max(np.abs(z.cpu().numpy() - z0)) <= 1e-13 * scale
        assert torch.equal(d.apply(xd), z)                # deterministic
        y = xd.clone()
        d.apply(y, y)                                     # z aliases r
        assert torch.equal(y, z)
        d.set_mode(1)                                     # resident sweep: same merged schedule, same bits
        assert torch.equal(d.apply(xd), z)
    monkeypatch.delenv("LG_IC0_MERGE")
    fm = L.ic0_factorize_multicolor(a)
    zm = fm.apply(x)
    Pm = fm.perm
    lm = fm.l
    zmr = np.empty(a.n)
    zmr[Pm] = O.Ic0(a.n, lm.row_ptr, lm.col_idx, lm.values).apply(x[Pm])
    assert np.max(np.abs(zm - zmr)) <= 1e-12 * np.max(np.abs(zmr))


@pytest.mark.parametrize("flags", [0, 1])
def test_gather_probe_runs(L, flags):
    """lg_spmv_gather_probe (the bench's gather floor) walks the stored column
    stream of either format without touching y; it must launch cleanly and
    leave x alone."""
    import torch
    from paper_1311_1695_b200.sparse import DeviceCsr
    a = L.build_laplacian(L.config_graph("C2"))
    d = DeviceCsr(a.n, a.row_ptr, a.col_idx, a.values, flags=flags)
    x = torch.randn(a.n, dtype=torch.float64, device="cuda")
    x0 = x.clone()
    d.gather_probe(x)
    torch.cuda.synchronize()
    assert torch.equal(x, x0)


def test_jacobi_variant(L):
    a = L.build_laplacian(L.config_graph("C1"))
    jf = L.JacobiFactor(a)
    x = np.random.default_rng(0).standard_normal(a.n)
    assert np.allclose(jf.apply(x), x / a.diagonal(), rtol=1e-15)


@pytest.mark.parametrize("cfg", ["C1", "C4"])
def test_plain_and_packed_formats_agree(L, cfg):
    import torch
    from paper_1311_1695_b200.sparse import DeviceCsr
    from paper_1311_1695_b200 import _device as dev
    a = L.build_laplacian(L.config_graph(cfg))
    plain = DeviceCsr(a.n, a.row_ptr, a.col_idx, a.values, flags=1)
    packed = DeviceCsr(a.n, a.row_ptr, a.col_idx, a.values)
    assert not plain.packed and packed.packed
    assert packed.stream_bytes < plain.stream_bytes
    x = torch.randn(a.n, dtype=torch.float64, device="cuda")
    y0, y1 = dev.empty(a.n), dev.empty(a.n)
    plain.matvec(x, y0, theta=0.3)
    packed.matvec(x, y1, theta=0.3)
    assert float((y0 - y1).abs().max()) <= 1e-13 * float(y0.abs().max())


@pytest.mark.parametrize("cfg", ["C2", "C3"])
def test_multicolor_ic0_variant(L, cfg):
    """Flagged variant: IC(0) of the colour-reordered matrix.  Its factor is
    the oracle's IC(0) of P A P^T bit for bit, the sweeps take #colours
    levels, and the apply (permutation folded into the sweeps) matches
    P^T (L L^T)^{-1} P r."""
    from paper_1311_1695_b200.ic0 import permuted_matrix
    a = L.build_laplacian(L.config_graph(cfg))
    f = L.ic0_factorize_multicolor(a)
    pa = permuted_matrix(a, f.perm)
    oa = O.Csr(a.n, pa.row_ptr, pa.col_idx, pa.values)
    lrp, lcol, lval, _, _ = O.ic0_factorize(oa, use_c=True)
    assert np.array_equal(f.l.values.view(np.int64), lval.view(np.int64))
    assert f.device().levels <= f.ncolors
    x = np.random.default_rng(0).standard_normal(a.n)
    zp = O.Ic0(a.n, lrp, lcol, lval).apply(x[f.perm])
    want = np.empty(a.n)
    want[f.perm] = zp
    z = f.apply(x)
    assert np.max(np.abs(z - want)) <= 1e-12 * np.max(np.abs(want))


def _download_i32(ptr, count):
    import ctypes
    from paper_1311_1695_b200 import _native as nat
    out = np.empty(count, dtype=np.int32)
    if count:
        nat.call("lg_readback", ptr, out.ctypes.data, 4 * count, None)
    return out


def test_device_rmat_lcc_laplacian_pipeline(L):
    """C5-scale ingest on the device, checked at scale 12 against the host
    pipeline: canonical edges, the same largest component, and an SpMV equal
    to the oracle's on the host-assembled Laplacian."""
    import ctypes
    from paper_1311_1695_b200 import _native as nat
    from paper_1311_1695_b200.device_graphs import DeviceLaplacian
    scale, ef = 12, 8
    di, dj, m = ctypes.c_void_p(), ctypes.c_void_p(), ctypes.c_int64()
    nat.call("lg_rmat_device", scale, ef, 0.57, 0.19, 0.19, ctypes.c_uint64(7),
             ctypes.byref(di), ctypes.byref(dj), ctypes.byref(m))
    n = 1 << scale
    i, j = _download_i32(di, m.value), _download_i32(dj, m.value)
    assert np.all(i < j)
    key = i.astype(np.int64) * n + j
    assert np.all(np.diff(key) > 0)
    g = L.graphs.EdgeList.from_canonical(n, i, j, np.ones(m.value))
    sub, _ = L.largest_component(g)
    nl, ml = ctypes.c_int64(), ctypes.c_int64()
    nat.call("lg_lcc_device", n, m.value, ctypes.byref(di), ctypes.byref(dj),
             ctypes.byref(nl), ctypes.byref(ml))
    assert (nl.value, ml.value) == (sub.n_nodes, sub.m)
    assert np.array_equal(_download_i32(di, ml.value), sub.i)
    assert np.array_equal(_download_i32(dj, ml.value), sub.j)
    h = ctypes.c_void_p()
    nat.call("lg_csr_laplacian_device", nl.value, ml.value, di, dj, ctypes.byref(h))
    nat.load().lg_free(di)
    nat.load().lg_free(dj)
    A = DeviceLaplacian(nl.value, ml.value, h)
    rp, col, val = O.build_laplacian(sub.n_nodes, sub.i, sub.j, sub.w)
    assert np.array_equal(A.diagonal(), O.Csr(sub.n_nodes, rp, col, val).dense().diagonal())
    x = np.random.default_rng(0).standard_normal(A.n)
    want = O.spmv(O.Csr(A.n, rp, col, val), x)
    y = L.spmv(A, x)
    assert np.max(np.abs(y - want)) <= 1e-13 * np.max(np.abs(want))
    # the host CSR of the device-only matrix (lg_csr_export_host: what the
    # host IC(0) factorization of a C5-family graph consumes) is the host
    # pipeline's Laplacian bit for bit, and so is its IC(0) factor
    erp = np.empty(A.n + 1, dtype=np.int64)
    ecol = np.empty(A.nnz, dtype=np.int64)
    evl = np.empty(A.nnz)
    nat.call("lg_csr_export_host", A.device().handle, erp.ctypes.data, ecol.ctypes.data,
             evl.ctypes.data)
    assert np.array_equal(erp, rp) and np.array_equal(ecol, col)
    assert np.array_equal(evl.view(np.int64), val.view(np.int64))
    f = L.ic0_factorize(L.CsrMatrix(A.n, erp, ecol, evl, symmetric=True))
    lrp, lcol, lval, _, _ = O.ic0_factorize(O.Csr(A.n, rp, col, val))
    assert np.array_equal(f.l.values.view(np.int64), lval.view(np.int64))


def test_csr_export_host_weighted(L):
    """lg_csr_export_host on host-built matrices: packed (integer weights,
    dense value table) and plain (real weights) both round-trip to the
    CsrMatrix arrays bit for bit."""
    from paper_1311_1695_b200 import _native as nat
    for g in (L.generators.chung_lu_graph(4000, 2.3, 6.0, weighted=True, seed=5),
              L.generators.random_connected_graph(3000, extra_edges=9000, seed=4,
                                                  weighted=True)):
        a = L.build_laplacian(g)
        rp = np.empty(a.n + 1, dtype=np.int64)
        col = np.empty(a.nnz, dtype=np.int64)
        val = np.empty(a.nnz)
        nat.call("lg_csr_export_host", a.device().handle, rp.ctypes.data, col.ctypes.data,
                 val.ctypes.data)
        assert np.array_equal(rp, a.row_ptr) and np.array_equal(col, a.col_idx)
        assert np.array_equal(val.view(np.int64), a.values.view(np.int64))


@pytest.mark.parametrize("world", [2, 3, 8])
def test_row_partitioned_spmv_row_blocks(L, world):
    """The multi-GPU SpMV's per-rank operators (the rank's rows, global
    columns, other rows absent from the schedule), run one after another on
    one device on the exchanged x, reproduce the single-device product to
    roundoff (a row block's warp windows need not fall where the full
    operator's do, so the per-row summation order may differ) and write only
    their own rows."""
    import torch
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.dist import RowPartition, local_operator
    a = L.build_laplacian(L.config_graph("C2"))
    part = RowPartition(a.row_ptr, world)
    x = torch.from_numpy(np.random.default_rng(4).standard_normal(a.n)).cuda()
    want = a.device()
    y_ref = dev.empty(a.n)
    want.matvec(x, y_ref)
    y = torch.zeros(a.n, dtype=torch.float64, device="cuda")
    for r in range(world):
        op = local_operator(a, part, r)
        assert op.packed == want.packed
        ys = torch.full((a.n,), 12345.0, dtype=torch.float64, device="cuda")
        op.matvec(x, ys)
        r0, r1 = part.rows(r)
        assert torch.all(ys[:r0] == 12345.0) and torch.all(ys[r1:] == 12345.0)
        y[r0:r1] = ys[r0:r1]
    assert float((y - y_ref).abs().max()) <= 1e-14 * float(y_ref.abs().max())


@pytest.mark.parametrize("world", [2, 5])
def test_row_partitioned_spmv_device_sliced(L, world):
    """Device-side row blocks of a device-only packed Laplacian (the C5 path:
    R-MAT sampled, LCC and assembled on the device) reproduce the full
    product to roundoff."""
    import torch
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import RowPartition, device_row_ptr, local_operator_device
    A = rmat_laplacian_device(13, 8, seed=3)
    full = A.device()
    part = RowPartition(device_row_ptr(full), world)
    x = torch.from_numpy(np.random.default_rng(5).standard_normal(A.n)).cuda()
    y_ref = dev.empty(A.n)
    full.matvec(x, y_ref)
    y = torch.zeros(A.n, dtype=torch.float64, device="cuda")
    for r in range(world):
        op = local_operator_device(full, part, r)
        ys = torch.full((A.n,), -7.0, dtype=torch.float64, device="cuda")
        op.matvec(x, ys)
        r0, r1 = part.rows(r)
        assert torch.all(ys[:r0] == -7.0) and torch.all(ys[r1:] == -7.0)
        y[r0:r1] = ys[r0:r1]
    assert float((y - y_ref).abs().max()) <= 1e-14 * float(y_ref.abs().max())


def test_spmv_host_buffers_cabi_and_public():
    """The host-buffer SpMV through the C ABI (lg_spmv_host: pinned staging,
    H2D, product, D2H) and through the public numpy spmv both equal the
    device product bit for bit, and match the oracle."""
    import ctypes

    import torch

    import paper_1311_1695_b200 as L
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200 import _native as nat
    # hubs above 1024 neighbours: the long-row path (needs the internal workspace)
    g, _ = L.largest_component(L.generators.chung_lu_graph(20000, 2.1, 8.0, max_degree=4000,
                                                           weighted=True, seed=11))
    a = L.build_laplacian(g)
    x = np.random.default_rng(3).standard_normal(a.n)
    yd = dev.empty(a.n)
    a.device().matvec(dev.to_device(x), yd)
    want = yd.cpu().numpy()
    y1 = L.spmv(a, x)
    assert np.array_equal(y1, want)
    y2 = np.empty(a.n)
    xd, ydd = dev.empty(a.n), dev.empty(a.n)
    nat.call("lg_spmv_host", a.device().handle, x.ctypes.data, y2.ctypes.data,
             ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(ydd.data_ptr()),
             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert np.array_equal(y2, want)
    yr = O.spmv(O.Csr(a.n, a.row_ptr, a.col_idx, a.values), x)
    assert np.max(np.abs(y2 - yr)) <= 1e-13 * np.max(np.abs(yr))
    # page-locked caller buffers are DMA'd directly (no staging)
    xp = torch.empty(a.n, dtype=torch.float64, pin_memory=True).numpy()
    yp = torch.empty(a.n, dtype=torch.float64, pin_memory=True).numpy()
    xp[:] = x
    nat.call("lg_spmv_host", a.device().handle, xp.ctypes.data, yp.ctypes.data,
             ctypes.c_void_p(xd.data_ptr()), ctypes.c_void_p(ydd.data_ptr()),
             ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert np.array_equal(yp, want)
    # every public product is a fresh array (pinned results are recycled
    # only after their array is gone)
    x2 = np.random.default_rng(4).standard_normal(a.n)
    keep = [L.spmv(a, x) for _ in range(3)]
    del y1
    y3 = L.spmv(a, x2)
    for k in keep:
        assert np.array_equal(k, want)
    assert not np.array_equal(y3, want)


@pytest.mark.parametrize("world", [2, 3])
def test_split_row_block_interior_exterior(world):
    """lg_csr_split_cols: a rank's row block = interior (own columns +
    diagonal) + exterior (every other column); inner product then
    lg_spmv_acc of the exterior equals the full product on the rank's rows
    (to roundoff: the two halves are summed separately) and leaves every
    other row untouched.  Host-built and device-built matrices."""
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200._plan import SpmvAcc
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import (RowPartition, local_operator_device, matrix_row_ptr,
                                           split_cols)
    g, _ = L.largest_component(L.generators.chung_lu_graph(20000, 2.1, 8.0, max_degree=4000,
                                                           weighted=True, seed=11))
    for A in (L.build_laplacian(g), rmat_laplacian_device(13, 8, seed=2)):
        full = A.device()
        n = A.n
        x = dev.to_device(np.random.default_rng(5).standard_normal(n))
        want = dev.empty(n)
        full.matvec(x, want)
        part = RowPartition(matrix_row_ptr(A), world)
        for r in range(world):
            r0, r1 = part.rows(r)
            op = local_operator_device(full, part, r)
            inner, outer = split_cols(op, r0, r1)
            assert inner.packed and outer.packed
            y = torch.full((n,), 777.0, dtype=torch.float64, device="cuda")
            inner.matvec(x, y)
            SpmvAcc(outer, x, y)()
            torch.cuda.synchronize()
            assert torch.all(y[:r0] == 777.0) and torch.all(y[r1:] == 777.0)
            err = (y[r0:r1] - want[r0:r1]).abs().max().item()
            assert err <= 1e-12 * max(1.0, want.abs().max().item())


@pytest.mark.parametrize("world", [2, 3])
def test_split_row_block_panelled_exterior(world):
    """The exterior half of a rank's row block as accumulating column panels
    (what C5's row-partitioned product uses: its x exceeds L2; forced here
    with LG_SPMV_PANELS=3 on small graphs): interior product + panelled
    exterior = the full product on the rank's rows to roundoff, every other
    row untouched; a panelled exterior refuses the non-accumulating lg_spmv."""
    import torch

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200._plan import SpmvAcc
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import (RowPartition, local_operator_device, matrix_row_ptr,
                                           split_cols)
    g, _ = L.largest_component(L.generators.chung_lu_graph(20000, 2.1, 8.0, max_degree=4000,
                                                           weighted=True, seed=13))
    for A in (L.build_laplacian(g), rmat_laplacian_device(13, 8, seed=4)):
        full = A.device()
        n = A.n
        x = dev.to_device(np.random.default_rng(6).standard_normal(n))
        want = dev.empty(n)
        full.matvec(x, want)
        part = RowPartition(matrix_row_ptr(A), world)
        for r in range(world):
            r0, r1 = part.rows(r)
            op = local_operator_device(full, part, r)
            os.environ["LG_SPMV_PANELS"] = "3"
            try:
                inner, outer = split_cols(op, r0, r1)
            finally:
                del os.environ["LG_SPMV_PANELS"]
            assert outer.npanels == 3
            y = torch.full((n,), 555.0, dtype=torch.float64, device="cuda")
            inner.matvec(x, y)
            SpmvAcc(outer, x, y)()
            torch.cuda.synchronize()
            assert torch.all(y[:r0] == 555.0) and torch.all(y[r1:] == 555.0)
            err = (y[r0:r1] - want[r0:r1]).abs().max().item()
            assert err <= 1e-12 * max(1.0, want.abs().max().item())
            with pytest.raises(ValueError):
                outer.matvec(x, y)


@pytest.mark.parametrize("panels", [2, 5])
def test_col_panels_sum_to_full_product(panels):
    """lg_csr_col_panel: the column panels of an operator (diagonal in the
    first) partition its nonzeros, and y = P_0 x, y += P_k x (lg_spmv_acc)
    equals the one-pass product to roundoff.  Host-built weighted and
    device-built R-MAT matrices."""
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200._plan import SpmvAcc
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import col_panel
    g, _ = L.largest_component(L.generators.chung_lu_graph(20000, 2.1, 8.0, max_degree=4000,
                                                           weighted=True, seed=11))
    for A in (L.build_laplacian(g), rmat_laplacian_device(13, 8, seed=2)):
        full = A.device()
        if not full.packed:
            continue
        n = A.n
        x = dev.to_device(np.random.default_rng(5).standard_normal(n))
        want = dev.empty(n)
        full.matvec(x, want)
        cuts = [n * k // panels for k in range(panels + 1)]
        parts = [col_panel(full, cuts[k], cuts[k + 1], k == 0) for k in range(panels)]
        assert sum(p.nnz for p in parts) == full.nnz
        y = dev.empty(n)
        parts[0].matvec(x, y)
        for p in parts[1:]:
            SpmvAcc(p, x, y)()
        err = (y - want).abs().max().item()
        assert err <= 1e-12 * max(1.0, want.abs().max().item())


def test_panelled_operator_solves_match():
    """lg_csr_set_panels: the panelled product (theta shift and epilogue
    dots included, as the solvers call it) gives the one-pass product to
    roundoff, and DACG / JD on a panelled operator return the same
    eigenvalues; detaching restores the one-pass product bitwise."""
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.precond import JacobiFactor
    A = rmat_laplacian_device(14, 8, seed=3)
    d = A.device()
    x = dev.to_device(np.random.default_rng(1).standard_normal(A.n))
    want, y, y2 = dev.empty(A.n), dev.empty(A.n), dev.empty(A.n)
    d.matvec(x, want, theta=0.37)
    f = JacobiFactor(A)
    ref_d, _ = L.dacg_smallest(A, 3, delta=1e-9, f=f, seed=0)
    ref_j, _ = L.jd_smallest(A, 3, delta=1e-9, f=f, seed=0)
    d.set_panels(3)
    try:
        d.matvec(x, y, theta=0.37)
        assert (y - want).abs().max().item() <= 1e-12 * want.abs().max().item()
        got_d, _ = L.dacg_smallest(A, 3, delta=1e-9, f=f, seed=0)
        got_j, _ = L.jd_smallest(A, 3, delta=1e-9, f=f, seed=0)
    finally:
        d.set_panels(0)
    assert np.max(np.abs(got_d.values - ref_d.values) / ref_d.values) <= 1e-8
    assert np.max(np.abs(got_j.values - ref_j.values) / ref_j.values) <= 1e-8
    d.matvec(x, y2, theta=0.37)
    assert bool((y2 == want).all())


def test_set_panels_rejects_row_blocks():
    """Column panels need a full operator: lg_csr_set_panels refuses a row
    block (host-built SKIP_EMPTY, or cut on the device), and LG_SPMV_PANELS
    never reaches a row block, so absent rows are still left untouched."""
    import os
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    from paper_1311_1695_b200.dist import (RowPartition, device_row_ptr, local_operator,
                                           local_operator_device)
    import paper_1311_1695_b200 as L
    a = L.build_laplacian(L.config_graph("C1"))
    part = RowPartition(a.row_ptr, 2)
    blk = local_operator(a, part, 1)
    with pytest.raises(ValueError, match="full operators"):
        blk.set_panels(2)
    A = rmat_laplacian_device(12, 8, seed=3)
    dblk = local_operator_device(A.device(), RowPartition(device_row_ptr(A.device()), 2), 0)
    with pytest.raises(ValueError, match="full operators"):
        dblk.set_panels(3)
    os.environ["LG_SPMV_PANELS"] = "3"
    try:
        blk2 = local_operator(a, part, 0)
    finally:
        del os.environ["LG_SPMV_PANELS"]
    assert blk2.npanels == 0
    r0, r1 = part.rows(0)
    x = dev.to_device(np.random.default_rng(2).standard_normal(a.n))
    y = dev.to_device(np.full(a.n, 7.0))
    blk2.matvec(x, y)
    assert bool((y[r1:] == 7.0).all())


def test_spmv_warp_schedule_edge_cases():
    """The warp-block schedule on the shapes that exercise each block kind:
    hub rows longer than a part (ticketed long-row parts), rows with no
    off-diagonal entry (row-serial blocks: isolated vertices outside an LCC,
    and rows of a SKIP_EMPTY operator), weighted values (value table), a plain
    (unpacked) matrix, rows that straddle lanes and the 16-byte window phase
    of every block start; each product matches the oracle's reduceat SpMV,
    theta-shifted and accumulating forms included, and is bitwise the same
    run to run."""
    import torch

    import paper_1311_1695_b200 as L
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.graphs import EdgeList
    rng = np.random.default_rng(7)
    cl = L.generators.chung_lu_graph(20000, 2.1, 8.0, max_degree=6000, weighted=True, seed=11)
    gs = [L.largest_component(cl)[0], cl, L.generators.star_graph(5000),
          L.generators.grid_graph(60, 70), L.generators.path_graph(3),
          L.generators.complete_graph(300)]
    for g in gs:
        a = L.build_laplacian(g)
        oa = O.Csr(a.n, a.row_ptr, a.col_idx, a.values)
        x = rng.standard_normal(a.n)
        want = O.spmv(oa, x)
        tol = 1e-13 * max(1.0, float(np.max(np.abs(want))))
        y = L.spmv(a, x)
        assert np.max(np.abs(y - want)) <= tol
        d = a.device()
        xd = dev.to_device(x)
        y1, y2 = dev.empty(a.n), dev.empty(a.n)
        d.matvec(xd, y1)
        d.matvec(xd, y2)
        assert torch.equal(y1, y2)
        yt = dev.empty(a.n)
        d.matvec(xd, yt, theta=0.75)
        assert np.max(np.abs(dev.to_host(yt) - (want - 0.75 * x))) <= tol
    # a plain-format operator: more distinct values than the packed table holds
    n = 3000
    i = rng.integers(0, n, 40000)
    j = rng.integers(0, n, 40000)
    keep = i != j
    lo, hi = np.minimum(i[keep], j[keep]), np.maximum(i[keep], j[keep])
    key = np.unique(lo.astype(np.int64) * n + hi)
    g = EdgeList(n, key // n, key % n, rng.random(key.size) + 0.5)
    a = L.build_laplacian(g)
    assert not a.device().packed
    x = rng.standard_normal(a.n)
    want = O.spmv(O.Csr(a.n, a.row_ptr, a.col_idx, a.values), x)
    assert np.max(np.abs(L.spmv(a, x) - want)) <= 1e-13 * np.max(np.abs(want))


@pytest.mark.gpu
@pytest.mark.parametrize("k", [2, 5, 8, 10, 16])
def test_spmm_rowmajor_matches_spmv(k):
    """lg_spmm_rowmajor (row-major X, one gather per nonzero for all k
    columns) equals k separate products to roundoff, hub rows (long-row
    parts) included; rayleigh_residuals through it agrees with the oracle's
    per-column residuals."""
    import torch

    import paper_1311_1695_b200 as L
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200 import _native as nat
    from paper_1311_1695_b200.results import rayleigh_residuals
    g, _ = L.largest_component(L.generators.chung_lu_graph(20000, 2.1, 8.0, max_degree=4000,
                                                           weighted=True, seed=11))
    a = L.build_laplacian(g)
    d = a.device()
    X = torch.as_tensor(np.random.default_rng(k).standard_normal((a.n, k)), device="cuda")
    Y = torch.empty_like(X)
    nat.call("lg_spmm_rowmajor", d.handle, X.data_ptr(), Y.data_ptr(), k,
             dev.workspace().handle, torch.cuda.current_stream().cuda_stream)
    for j in range(k):
        yj = dev.empty(a.n)
        d.matvec(X[:, j].contiguous(), yj)
        torch.cuda.synchronize()
        assert (Y[:, j] - yj).abs().max().item() <= 1e-12 * max(1.0, yj.abs().max().item())
    V = np.random.default_rng(1).standard_normal((a.n, k))
    th, res = rayleigh_residuals(a, V)
    oa = O.Csr(a.n, a.row_ptr, a.col_idx, a.values)
    th_o, res_o = O.rayleigh_residuals(oa, V)
    assert np.allclose(th, th_o, rtol=1e-12) and np.allclose(res, res_o, rtol=1e-10)


@pytest.mark.parametrize("m,p", [(0, 3), (5, 1), (60, 20), (120, 51), (64, 32), (7, 70)])
def test_gemm_small_any_shape(m, p):
    """lg_gemm_small tiles any (m, p): IRLM's Ritz vectors at neig 20
    (ncv 60) and 50 (ncv 120) exceed one 64 x 32 / 1024-entry tile (the
    reference's acceptance criterion 1 runs neig 20, test_acceptance.py:102)."""
    import ctypes
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200 import _native as nat
    n = 1000
    rng = np.random.default_rng(m * 100 + p)
    src = rng.standard_normal((max(m, 1), n))
    y = np.asfortranarray(rng.standard_normal((m, p)))
    sd, out = dev.to_device(src), dev.to_device(np.full((p, n), 3.0))
    nat.call("lg_gemm_small", n, sd.data_ptr(), n, m, y.ctypes.data if m else None, p,
             out.data_ptr(), n, ctypes.c_void_p(dev.stream_ptr()))
    want = (src[:m].T @ y).T
    got = dev.to_host(out)
    assert np.max(np.abs(got - want)) <= 1e-12 * max(1.0, np.max(np.abs(want)))
