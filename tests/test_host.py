"""Host-side logic that needs no GPU: the C ABI library loads and exports
its header, the bit-exact host IC(0) factorization, input validation that
mirrors the reference, generators, and the no-fallback guarantee."""

import hashlib
import re
from pathlib import Path

import numpy as np
import pytest

from tests.conftest import ROOT, cuda_ok, golden_config, kat_edges


def header_symbols():
    text = (ROOT / "include" / "lapb200.h").read_text()
    return sorted(set(re.findall(r"^\s*(?:int|const char\*)\s+(lg_\w+)\(", text, re.M)))


def test_library_exports_every_header_symbol():
    import ctypes
    from paper_1311_1695_b200 import _native
    lib = _native.load()
    syms = header_symbols()
    assert len(syms) >= 20
    for s in syms:
        assert hasattr(lib, s), f"{s} missing from liblapb200.so"
    assert set(syms) == set(_native.EXPORTED)
    assert lib.lg_version() >= 100
    assert isinstance(ctypes.CDLL(str(_native.LIB_PATH)), ctypes.CDLL)


def test_library_is_sm100a():
    import subprocess
    from paper_1311_1695_b200 import _native
    out = subprocess.run(["cuobjdump", "--list-elf", str(_native.LIB_PATH)],
                         capture_output=True, text=True)
    if out.returncode != 0:
        pytest.skip("cuobjdump unavailable")
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("name", ["P4", "grid4x5", "rand50", "rand200", "geo1000"])
def test_host_ic0_factor_bit_exact(kat, name):
    """lg_ic0_factorize (host C++) reproduces the reference factor bit for bit."""
    from paper_1311_1695_b200.ic0 import ic0_factorize
    from paper_1311_1695_b200.sparse import CsrMatrix
    graphs, arrays, results = kat
    n = int(graphs[name + "_n"][0])
    a = CsrMatrix(n, arrays[name + "_rp"], arrays[name + "_col"], arrays[name + "_val"],
                  symmetric=True)
    f = ic0_factorize(a)
    assert np.array_equal(f.l.row_ptr, arrays[name + "_lrp"])
    assert np.array_equal(f.l.col_idx, arrays[name + "_lcol"])
    assert np.array_equal(f.l.values.view(np.int64), arrays[name + "_lval"].view(np.int64))
    assert f.shift == results[name]["ic0_shift"]


@pytest.mark.parametrize("cfg", ["C1", "C2"])
def test_host_ic0_factor_configs(cfg):
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.generators import config_graph
    from paper_1311_1695_b200.ic0 import ic0_factorize
    from paper_1311_1695_b200.sparse import CsrMatrix
    ref = golden_config(cfg)
    g = config_graph(cfg)
    rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    f = ic0_factorize(CsrMatrix(g.n_nodes, rp, col, val, symmetric=True))
    h = hashlib.sha256()
    for x in (f.l.row_ptr, f.l.col_idx, f.l.values):
        h.update(np.ascontiguousarray(x).tobytes())
    assert h.hexdigest() == ref["ic0_sha256"]


@pytest.mark.parametrize("name", ["P4", "grid4x5", "rand50", "rand200", "geo1000", "C1", "C2"])
def test_level_merged_system_solves_like_the_factor(kat, name):
    """Host half of the device IC(0) apply: the level-merged system (auxiliary
    partial sums, the level below substituted, right-hand-side entries; any
    number of passes) solved in its own topological order gives the plain
    triangular solves of ic0.py:40-45 to roundoff, with a shallower DAG."""
    import ctypes
    import scipy.sparse as sp
    import scipy.sparse.linalg as spla
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200 import _native as nat
    from paper_1311_1695_b200.generators import config_graph
    from paper_1311_1695_b200.ic0 import ic0_factorize
    from paper_1311_1695_b200.sparse import CsrMatrix
    if name.startswith("C"):
        g = config_graph(name)
        rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
        a = CsrMatrix(g.n_nodes, rp, col, val, symmetric=True)
    else:
        graphs, arrays, _ = kat
        a = CsrMatrix(int(graphs[name + "_n"][0]), arrays[name + "_rp"], arrays[name + "_col"],
                      arrays[name + "_val"], symmetric=True)
    l = ic0_factorize(a).l
    n = l.n
    lrp = np.ascontiguousarray(l.row_ptr, dtype=np.int64)
    lcol = np.ascontiguousarray(l.col_idx, dtype=np.int64)
    lval = np.ascontiguousarray(l.values, dtype=np.float64)
    Lm = sp.csr_matrix((lval, lcol, lrp), shape=(n, n))
    b = np.random.default_rng(7).standard_normal(n)
    want = {0: spla.spsolve_triangular(Lm, b, lower=True),
            1: spla.spsolve_triangular(Lm.T.tocsr(), b, lower=False)}
    for backward in (0, 1):
        depth0 = None
        for passes in (0, 1, 2, 4):
            y = np.empty(n)
            dep, ent, unk = ctypes.c_int(), ctypes.c_int64(), ctypes.c_int64()
            nat.call("lg_ic0_merged_solve_host", n, lrp.ctypes.data, lcol.ctypes.data,
                     lval.ctypes.data, passes, backward, b.ctypes.data, y.ctypes.data,
                     ctypes.byref(dep), ctypes.byref(ent), ctypes.byref(unk))
            ref = want[backward]
            assert np.max(np.abs(y - ref)) <= 1e-12 * np.max(np.abs(ref)), (backward, passes)
            if passes == 0:
                depth0 = dep.value
                assert ent.value == lrp[-1] - n and unk.value == n
            else:
                assert dep.value <= depth0 and unk.value >= n and ent.value >= lrp[-1] - n
                if depth0 >= 8:
                    assert dep.value < depth0                # a real chain gets shorter


def test_ic0_shift_ladder_and_breakdown():
    from paper_1311_1695_b200.ic0 import Ic0Error, ic0_factorize
    from paper_1311_1695_b200.sparse import CsrMatrix
    # an indefinite symmetric matrix: every shift fails until 0.1 * max diag
    dense = np.array([[1.0, 1.05], [1.05, 1.0]])
    r, c = np.nonzero(dense)
    a = CsrMatrix.from_coo(2, r, c, dense[r, c], symmetric=True)
    f = ic0_factorize(a)
    assert f.attempts == 7 and f.shift == pytest.approx(0.1)
    f2 = ic0_factorize(a, shift0=0.2)
    assert f2.attempts == 1 and f2.shift == 0.2
    neg = CsrMatrix.from_coo(2, [0, 1], [0, 1], [-1.0, -1.0], symmetric=True)
    with pytest.raises(Ic0Error):
        ic0_factorize(neg)
    with pytest.raises(ValueError):
        ic0_factorize(CsrMatrix.identity(3).__class__(3, [0, 1, 2, 3], [0, 1, 2], [1, 1, 1]))


def test_csr_validation_mirrors_reference():
    from paper_1311_1695_b200.sparse import CsrMatrix, MvpCounter
    with pytest.raises(ValueError):
        CsrMatrix(2, [0, 1], [0], [1.0])
    with pytest.raises(ValueError):
        CsrMatrix(2, [1, 1, 2], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        CsrMatrix(2, [0, 2, 1], [0, 1], [1.0, 1.0])
    with pytest.raises(ValueError):
        CsrMatrix(2, [0, 2, 2], [1, 0], [1.0, 1.0])
    with pytest.raises(ValueError):
        CsrMatrix(2, [0, 1, 2], [0, 5], [1.0, 1.0])
    with pytest.raises(ValueError):
        CsrMatrix.from_coo(2, [0, 0], [1, 1], [1.0, 2.0])
    a = CsrMatrix.from_coo(3, [2, 0, 1], [0, 2, 1], [1.0, 2.0, 3.0])
    assert a.nnz == 3 and np.allclose(a.toarray(), [[0, 0, 2], [0, 3, 0], [1, 0, 0]])
    assert np.allclose(a.diagonal(), [0, 3, 0])
    c = MvpCounter()
    c.increment()
    c.increment(4)
    assert c.count == 5 and "5" in repr(c)


def test_edgelist_canonicalisation_and_errors():
    from paper_1311_1695_b200.graphs import EdgeList
    g = EdgeList(4, [3, 1, 0], [1, 2, 2], [1.0, 2.0, 3.0])
    assert g.i.tolist() == [0, 1, 1] and g.j.tolist() == [2, 2, 3]
    for bad in ([(0, 0, 1.0)], [(0, 1, 0.0)], [(0, 1, 1.0), (1, 0, 2.0)], [(0, 9, 1.0)]):
        with pytest.raises(ValueError):
            EdgeList.from_pairs(4, bad)
    with pytest.raises(ValueError):
        EdgeList(0, [], [], [])


def test_components_and_lcc():
    from paper_1311_1695_b200.graphs import EdgeList, connected_components, largest_component
    g = EdgeList(7, [0, 1, 3, 4, 5], [1, 2, 4, 5, 6], np.ones(5))
    count, labels = connected_components(g)
    assert count == 2 and labels[0] == 0 and labels[3] == 1
    sub, node_map = largest_component(g)
    assert sub.n_nodes == 4 and node_map[0] == -1 and node_map[3] == 0


def test_generators_match_baseline_sizes():
    from paper_1311_1695_b200.generators import config_graph
    for cfg in ("C1", "C2"):
        ref = golden_config(cfg)
        g = config_graph(cfg)
        assert (g.n_nodes, g.m) == (ref["n"], ref["m"])


def test_dense_eig_and_ncv():
    from paper_1311_1695_b200.irlm import ncv_for
    from paper_1311_1695_b200.kernels import dense_sym_eig, tridiag_eig
    rng = np.random.default_rng(0)
    h = rng.standard_normal((6, 6))
    h = h + h.T
    w, v = dense_sym_eig(h)
    assert np.allclose(w, np.linalg.eigvalsh(h)) and np.allclose(v.T @ v, np.eye(6))
    with pytest.raises(ValueError):
        dense_sym_eig(np.triu(h) + 1.0)
    with pytest.raises(ValueError):
        dense_sym_eig(np.eye(3), max_dim=2)
    w, _ = tridiag_eig([2.0, 2.0, 2.0], [-1.0, -1.0])
    assert np.allclose(w, 2 - 2 * np.cos(np.pi * np.arange(1, 4) / 4))
    assert [ncv_for(k) for k in (1, 5, 20, 50, 60)] == [15, 30, 60, 120, 140]
    with pytest.raises(ValueError):
        ncv_for(0)


def test_deflation_basis_validation():
    from paper_1311_1695_b200.pcg import DeflationBasis, kernel_basis
    with pytest.raises(ValueError):
        DeflationBasis(np.ones((4, 2)))
    with pytest.raises(ValueError):
        DeflationBasis.single(np.zeros(3))
    kb = kernel_basis(5, labels=np.array([0, 0, 1, 1, 1]))
    assert kb.k == 2 and np.allclose(kb.columns[:2, 0], 1 / np.sqrt(2))
    assert np.allclose(kernel_basis(4).columns[:, 0], 0.5)


@pytest.mark.skipif(cuda_ok(), reason="checks the no-GPU failure mode")
def test_no_cpu_fallback():
    """Every compute entry point raises without a CUDA device."""
    from paper_1311_1695_b200.sparse import CsrMatrix, spmv
    a = CsrMatrix.identity(3)
    with pytest.raises(RuntimeError):
        spmv(a, np.ones(3))
    from paper_1311_1695_b200.graphs import EdgeList, build_laplacian
    with pytest.raises(RuntimeError):
        build_laplacian(EdgeList(2, [0], [1], [1.0]))


def test_row_partitioned_pass_addresses():
    """The plan context of a row-partitioned rank (_plan.Ctx): every pass
    covers exactly the rank's rows of the full-length buffers (vectors and
    column blocks offset by 8 r0 bytes, block leading dimension n), a pass
    with dot products is followed by one all-reduce of its result slots and
    then its scalar program, and a single rank folds nothing (no GPU needed:
    the launches are only built)."""
    import torch

    from paper_1311_1695_b200._plan import AllReduce, Ctx, Fused, Seq

    class FakeComm:
        world, r0, r1 = 3, 100, 250
        nl = 150

        def __init__(self):
            self.reduced = []

        def allreduce_(self, t):
            self.reduced.append(t.numel())

    n, k = 400, 3
    x, y = torch.zeros(n, dtype=torch.float64), torch.zeros(n, dtype=torch.float64)
    C = torch.zeros((k, n), dtype=torch.float64)
    res = torch.zeros(16, dtype=torch.float64)
    comm = FakeComm()
    cx = Ctx(n, comm)
    assert cx.dist and cx.lo == 100 and cx.nl == 150
    seq = cx.fused(outs=[dict(out=y, terms=[(x, 2.0)], upd=(C, k, 0))],
                   dots=[(1, x)], blocks=[(C, k, 1)], result=res)
    assert isinstance(seq, Seq) and isinstance(seq.steps[1], AllReduce)
    f = seq.fused
    a = f.args
    assert a.n == 150
    assert a.o[0].out == y.data_ptr() + 800 and a.o[0].t[0].v == x.data_ptr() + 800
    assert a.o[0].uq == C.data_ptr() + 800 and a.o[0].uld == n and a.o[0].uk == k
    assert a.db[0] == x.data_ptr() + 800
    assert a.b[0].q == C.data_ptr() + 800 and a.b[0].ld == n and a.b[0].k == k
    seq.steps[1]()
    assert comm.reduced == [1 + k]          # one all-reduce over dots + Q^T v slots
    # one rank: the plain single-GPU pass, nothing wrapped
    one = Ctx(n, None).fused(dots=[(x, None)], result=res)
    assert isinstance(one, Fused) and one.args.n == n


def _fsai_numpy(n, rp, col, val, kmax):
    """Test-side restatement of the FSAI rows (lg_fsai.cu): pattern = the
    strictly lower columns cut to kmax - 1 by |a_ij| (ties to larger j) plus
    the diagonal; A[P, P] g = e_last; row = g / sqrt(g_last)."""
    import numpy.linalg as la
    A = np.zeros((n, n))
    for r in range(n):
        A[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
    G = np.zeros((n, n))
    for i in range(n):
        c, v = col[rp[i]:rp[i + 1]], val[rp[i]:rp[i + 1]]
        low = [(abs(x), j) for j, x in zip(c, v) if j < i]
        low.sort(key=lambda t: (-t[0], -t[1]))
        P = sorted(j for _, j in low[:kmax - 1]) + [i]
        e = np.zeros(len(P))
        e[-1] = 1.0
        g = la.solve(A[np.ix_(P, P)], e)
        G[i, P] = g / np.sqrt(g[-1])
    return A, G


@pytest.mark.parametrize("kmax", [4, 64])
def test_fsai_factor_rows(kmax):
    """lg_fsai_factorize (host C++) against the restatement, and the FSAI
    property diag(G A G^T) = 1 (no GPU needed)."""
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.generators import chung_lu_graph
    from paper_1311_1695_b200.graphs import largest_component
    from paper_1311_1695_b200.precond import FsaiFactor
    from paper_1311_1695_b200.sparse import CsrMatrix
    g, _ = largest_component(chung_lu_graph(300, 2.1, 5.0, max_degree=60, weighted=True, seed=4))
    rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    a = CsrMatrix(g.n_nodes, rp, col, val)
    f = FsaiFactor(a, kmax=kmax)
    n = a.n
    A, Gw = _fsai_numpy(n, rp, col, val, kmax)
    G = np.zeros((n, n))
    for r in range(n):
        G[r, f.g.col_idx[f.g.row_ptr[r]:f.g.row_ptr[r + 1]]] = \
            f.g.values[f.g.row_ptr[r]:f.g.row_ptr[r + 1]]
    assert np.array_equal(G != 0, Gw != 0)
    assert np.max(np.abs(G - Gw)) <= 1e-11 * np.max(np.abs(Gw))
    assert np.allclose(np.diag(G @ A @ G.T), 1.0, atol=1e-10)
    GT = np.zeros((n, n))
    for r in range(n):
        GT[r, f.gt.col_idx[f.gt.row_ptr[r]:f.gt.row_ptr[r + 1]]] = \
            f.gt.values[f.gt.row_ptr[r]:f.gt.row_ptr[r + 1]]
    assert np.array_equal(GT, G.T)


def test_graph_loader_matches_reference_cases():
    """load_edge_list (C++ lg_graph_parse) on the golden inputs: the same
    canonical edge list (bitwise weights) or the same GraphFormatError
    message and line as the reference's parsers (graphs.py:126-247;
    tests/golden/make_loader_golden.py ran them)."""
    import json

    import paper_1311_1695_b200 as L
    cases = json.loads((Path(__file__).parent / "golden" / "loader_cases.json").read_text())
    for rec in cases:
        src = rec["text"].encode()
        if "error" in rec:
            with pytest.raises(L.GraphFormatError) as err:
                L.load_edge_list(src, format=rec["format"], symmetrize=rec["symmetrize"])
            assert str(err.value) == rec["error"], (rec["text"], str(err.value))
            assert err.value.line == rec["line"]
        else:
            g = L.load_edge_list(src, format=rec["format"], symmetrize=rec["symmetrize"])
            assert g.n_nodes == rec["n"]
            assert g.i.tolist() == rec["i"] and g.j.tolist() == rec["j"]
            assert [float(x).hex() for x in g.w] == rec["w"]


def test_graph_loader_paths_streams_and_round_trip(tmp_path):
    """Paths, text streams and bytes give the same graph; Matrix Market
    output of a Laplacian reads back as the same graph (graphs.py:347-361);
    stats and csr_connected_components count components."""
    import io

    import paper_1311_1695_b200 as L
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.sparse import CsrMatrix
    text = "6\n0 1 1.5\n1 2 2\n# gap\n3 4 0.5\n"
    p = tmp_path / "g.txt"
    p.write_text(text)
    a = L.load_edge_list(str(p))
    b = L.load_edge_list(io.StringIO(text))
    c = L.load_edge_list(text.encode())
    assert a.pairs() == b.pairs() == c.pairs() == [(0, 1, 1.5), (1, 2, 2.0), (3, 4, 0.5)]
    st = L.stats(a)
    assert (st.n, st.nnz, st.components) == (6, 12, 3)
    rp, col, val = O.build_laplacian(a.n_nodes, a.i, a.j, a.w)
    lap = CsrMatrix(a.n_nodes, rp, col, val, symmetric=True)
    blob = L.write_matrix_market(lap)
    back = L.load_edge_list(blob.encode(), format="mtx")
    assert back.pairs() == a.pairs()
    count, labels = L.csr_connected_components(lap)
    assert count == 3 and labels.tolist() == [0, 0, 0, 1, 1, 2]
    with pytest.raises(ValueError):
        L.load_edge_list(b"", format="csv")


def test_fsai2_pattern_and_rows():
    """FSAI(2) (levels=2): each row's pattern is the kmax - 1 best lower
    candidates by |a_ij| + sum_k |a_ik||a_kj| (k: neighbours with at most
    64 entries), ties to the larger column, plus the diagonal; the rows solve
    A[P, P] g = e_last (diag(G A G^T) = 1)."""
    from oracle import lapeig_oracle as O
    from paper_1311_1695_b200.generators import chung_lu_graph
    from paper_1311_1695_b200.graphs import largest_component
    from paper_1311_1695_b200.precond import FsaiFactor
    from paper_1311_1695_b200.sparse import CsrMatrix
    g, _ = largest_component(chung_lu_graph(400, 2.1, 5.0, max_degree=80, weighted=True, seed=8))
    rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    a = CsrMatrix(g.n_nodes, rp, col, val)
    n, kmax = a.n, 8
    f = FsaiFactor(a, kmax=kmax, levels=2)
    A = np.zeros((n, n))
    for r in range(n):
        A[r, col[rp[r]:rp[r + 1]]] = val[rp[r]:rp[r + 1]]
    deg = np.diff(rp)
    for i in range(n):
        score = {}
        for q in range(rp[i], rp[i + 1]):
            k = col[q]
            if k == i:
                continue
            if k < i:
                score[k] = score.get(k, 0.0) + abs(val[q])
            if deg[k] > 64:
                continue
            for t in range(rp[k], rp[k + 1]):
                j = col[t]
                if j < i and j != k:
                    score[j] = score.get(j, 0.0) + abs(val[q]) * abs(val[t])
        best = sorted(score.items(), key=lambda kv: (-kv[1], -kv[0]))[:kmax - 1]
        P = sorted(j for j, _ in best) + [i]
        got = f.g.col_idx[f.g.row_ptr[i]:f.g.row_ptr[i + 1]].tolist()
        assert got == P, (i, got, P)
        e = np.zeros(len(P))
        e[-1] = 1.0
        gw = np.linalg.solve(A[np.ix_(P, P)], e)
        gw /= np.sqrt(gw[-1])
        gv = f.g.values[f.g.row_ptr[i]:f.g.row_ptr[i + 1]]
        assert np.max(np.abs(gv - gw)) <= 1e-10 * np.max(np.abs(gw))


def test_bench_arms_print_the_same_config():
    """bench.py's two arms (the B200 product and --impl reference) print the
    same `config` object for a workload, so the driver can pair their lines;
    and the reference arm's JSON line carries the contract's keys."""
    import importlib.util
    import json
    import subprocess
    import sys
    spec = importlib.util.spec_from_file_location("bench_mod", ROOT / "bench.py")
    bench = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(bench)
    c1 = bench.bench_config("C4", 989777, 10907457, 1)
    c2 = bench.bench_config("C4", 989777, 10907457, 1)
    assert c1 == c2 and c1["n"] == 989777 and "workload" in c1
    out = subprocess.run([sys.executable, str(ROOT / "bench.py"), "--impl", "reference",
                          "--config", "C1", "--steps", "3", "--warmup", "3"],
                         capture_output=True, text=True, timeout=600, cwd=str(ROOT))
    assert out.returncode == 0, out.stderr[-2000:]
    line = json.loads(out.stdout.strip().splitlines()[-1])
    assert line["impl"] == "reference" and line["unit"] == "matvecs/s"
    assert line["config"] == bench.bench_config("C1", line["config"]["n"],
                                                 line["config"]["nnz"], 1)
    assert line["e2e"]["h2d_bytes_per_step"] == 0 and line["cpu_baseline"]["kind"] == "port"
