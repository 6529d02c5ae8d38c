"""Per-pass roofline of one DACG iteration (SURVEY 8(d) "One DACG
iteration"), dev aid behind profiles/r02_dacg_iter_roofline.json.

Builds the device DACG plan on a config graph (reference IC(0), or FSAI with
--fsai) mid-solve (deflation basis of k columns: the kernel vector plus
k - 1 orthonormal ones), then for every launch of one iteration:
  * algorithmic bytes: 8 n for every distinct n-vector the pass reads or
    writes (operands aliased to the pass's own outputs are not re-read),
    8 n per Q column of a block dot / update; the SpMV's stream bytes
    (lg_csr_info); the IC(0) apply's SURVEY model
    B_ic0 = 2 (12 nnz_L + 8 (n+1)) + 32 n;
  * device time: CUDA events around the launch alone, L2 flushed before it
    (256 MiB write, untimed), median of 20;
and the whole iteration (CUDA graph, no flush) against the SURVEY model
B_spmv + B_ic0 + 2 (2k+3) 8n + 10 8n.
usage: python scripts/iter_roofline.py [C4] [--k 6] [--fsai]"""
import json
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200._plan import Fused, PrecApply, Seq, Spmv  # noqa: E402
from paper_1311_1695_b200.dacg import _DacgPlan  # noqa: E402

cfg = next((x for x in sys.argv[1:] if not x.startswith("--") and not x.isdigit()), "C4")
k = int(sys.argv[sys.argv.index("--k") + 1]) if "--k" in sys.argv else 6
peak = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())["hbm_gbs"] \
    if (ROOT / "MEASURED_PEAKS.json").exists() else 6535.1

a = L.build_laplacian(L.config_graph(cfg))
f = L.fsai_factorize(a, kmax=32) if "--fsai" in sys.argv else L.ic0_factorize(a)
n = a.n
nnz_l = (a.nnz + n) // 2
B_ic0 = 2 * (12 * nnz_l + 8 * (n + 1)) + 32 * n


def fused_bytes(fz):
    A = fz.args
    reads, writes, qcols = set(), set(), 0
    for o in A.o:
        if not o.out:
            continue
        writes.add(o.out)
        for t in range(o.nterms):
            v = o.t[t].v
            if v and v > 3:
                reads.add(v)
        qcols += max(o.uk, 0) + max(o.uk2, 0)
    for d in range(A.ndots):
        for v in (A.da[d], A.db[d], A.dc[d]):
            if v and v > 3:
                reads.add(v)
    for b in range(A.nblocks):
        qcols += A.b[b].k
        if A.b[b].v and A.b[b].v > 3:
            reads.add(A.b[b].v)
    reads -= writes   # an output re-read by the same pass is not streamed twice
    return 8 * n * (len(reads) + len(writes) + qcols), len(reads), len(writes), qcols


def flat(steps):
    out = []
    for s in steps:
        out += flat(s.steps) if isinstance(s, Seq) else [s]
    return out


def ev(fn, flush=None, reps=20):
    st = torch.cuda.current_stream()
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        if flush is not None:
            flush.fill_(1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        fn()
        e1.record(st)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1) * 1e3)
    return float(np.median(ts))


with dev.solver_stream():
    pl = _DacgPlan(a, f, n, 11)
    Qm = np.linalg.qr(np.column_stack([np.ones(n)] + [np.random.default_rng(j).standard_normal(n)
                                                      for j in range(k - 1)]))[0]
    for j in range(k):
        pl.C[j] = torch.from_numpy(np.ascontiguousarray(Qm[:, j])).cuda()
    pl.k = k
    x = dev.to_device(np.random.default_rng(0).standard_normal(n))
    pl.X[0].copy_(x / x.norm())
    pl.X[1].copy_(pl.X[0])
    Spmv(pl.csr, pl.X[0], pl.AX[0])()
    pl.AX[1].copy_(pl.AX[0])
    pl.G[0].copy_(pl.AX[0])
    pl.G[1].copy_(pl.AX[0])
    pl.P.zero_()
    pl.S.set(since=10, period=100, q=1.0, delta=-1.0)   # never a convergence halt
    steps = flat(pl.plan(0))
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    rows, tot_b, tot_t = [], 0, 0.0
    for i, fn in enumerate(steps):
        def run(fn=fn):
            pl.p_clear()
            fn()
        us = ev(run, flush)
        if isinstance(fn, Fused):
            b, nr, nw, qc = fused_bytes(fn)
            what = f"fused pass: {nr} vectors read, {nw} written, {qc} Q columns"
        elif isinstance(fn, Spmv):
            b = fn.csr.stream_bytes
            what = "SpMV (packed stream + schedule + diagonal + x + y)"
        elif isinstance(fn, PrecApply):
            b = B_ic0 if not "--fsai" in sys.argv else None
            what = "IC(0) apply (SURVEY B_ic0)" if b else "FSAI apply (2 SpMVs)"
            if b is None:
                b = 2 * 12 * int(f.g.nnz) + 2 * 24 * n if hasattr(f, "g") else 0
        else:
            b, what = 0, type(fn).__name__
        rows.append({"launch": i, "kind": type(fn).__name__, "what": what, "bytes": int(b),
                     "us_l2_flushed": round(us, 2),
                     "gbs": round(b / (us * 1e-6) / 1e9, 1) if b and us else None,
                     "frac_of_peak": round(b / (us * 1e-6) / 1e9 / peak, 3) if b and us else None})
        tot_b += b
        tot_t += us
    g = pl.graph(0)
    for _ in range(3):
        pl.p_clear()
        g()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(100):
        pl.p_clear()
        g()
    e1.record(st)
    torch.cuda.synchronize()
    it_us = e0.elapsed_time(e1) / 100 * 1e3

B_spmv = 12 * a.nnz + 8 * (n + 1) + 16 * n
model = B_spmv + B_ic0 + 2 * (2 * k + 3) * 8 * n + 10 * 8 * n
out = {"config": cfg, "n": n, "nnz": a.nnz, "k": k,
       "preconditioner": "fsai kmax 32" if "--fsai" in sys.argv else "ic0 (reference)",
       "peak_gbs": peak, "launches": rows,
       "sum_of_isolated_us": round(tot_t, 1), "sum_bytes": int(tot_b),
       "iteration_graph_us": round(it_us, 1),
       "survey_model_bytes": int(model),
       "survey_model_gbs": round(model / (it_us * 1e-6) / 1e9, 1),
       "survey_model_frac": round(model / (it_us * 1e-6) / 1e9 / peak, 3),
       "executed_bytes_gbs": round(tot_b / (it_us * 1e-6) / 1e9, 1)}
print(json.dumps(out))
