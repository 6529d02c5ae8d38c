"""Benchmark: Laplacian SpMV GB/s & matvecs/s, and wall time to k smallest
eigenpairs (DACG / JD), on the BASELINE configuration C4 (weighted
Chung-Lu, n = 1e6, power-law exponent 2.5, mean degree 10, Geometric(0.5)
integer weights, largest component: n = 989,777, nnz = 10,907,457).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--config C4] [--no-solve]

A "step" is one Laplacian matvec y = L x of the whole graph.  value is
matvecs/s of the fused device SpMV with inputs resident in HBM (L2 flushed
between steps by writing a 256 MiB buffer outside the timed events); e2e is
the same metric through the public API spmv(a, x) with host numpy buffers
(H2D of x + D2H of y inside the timed region).  roofline uses the SURVEY
8(d) byte model (12 nnz + 8 (n+1) + 16 n per matvec) against the measured
HBM copy bandwidth in MEASURED_PEAKS.json.  cpu_baseline times the oracle's
restatement of the reference SpMV (np.add.reduceat per row,
sparse.py:128-139) on this host.  The solve block reports DACG and JD wall
time to 5 eigenpairs at delta = 1e-8 (the configuration of the reference
runs recorded in tests/golden/config_C4.json).

With N > 1 (torchrun, one rank per GPU) the matrix is row-partitioned by
nonzeros; every step all-gathers x over NCCL and multiplies the local row
block (strong scaling: the whole-job value is matvecs/s of the global
matrix, timed as the max over ranks).

--impl reference runs the CPU reference arm: the oracle's restatement of the
reference SpMV, row-chunked over all host threads, on rank 0 only.
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "Laplacian SpMV matvecs/s (C4 weighted Chung-Lu 1M); wall time to k eigenpairs"
UNIT = "matvecs/s"


def _peaks():
    try:
        return json.loads((ROOT / "MEASURED_PEAKS.json").read_text()), "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}, "fallback"


class ClockSampler:
    """nvidia-smi clocks / throttle reasons sampled during the timed region."""

    FIELDS = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = None
        self.source = "nvidia-smi"
        # in-process NVML when available: a query takes tens of microseconds, so
        # a timed region of a few milliseconds still gets several samples taken
        # while it runs (an nvidia-smi process takes ~50 ms to come back)
        self._nvml = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self._nvml = pynvml
            self.source = "nvml"
        except Exception:
            self._nvml = None

    def _sample_nvml(self):
        n = self._nvml
        sm = n.nvmlDeviceGetClockInfo(self._h, n.NVML_CLOCK_SM)
        mx = n.nvmlDeviceGetMaxClockInfo(self._h, n.NVML_CLOCK_SM)
        get = getattr(n, "nvmlDeviceGetCurrentClocksEventReasons", None) or getattr(
            n, "nvmlDeviceGetCurrentClocksThrottleReasons")
        bits = int(get(self._h))
        # NVML reason bits: HwSlowdown 0x8, HwThermalSlowdown 0x40,
        # SwThermalSlowdown 0x20, SwPowerCap 0x4
        flags = ["Active" if bits & b else "Not Active" for b in (0x8, 0x40, 0x20, 0x4)]
        return [str(sm), str(mx)] + flags

    def _run(self):
        while not self._stop.is_set():
            if self._nvml is not None:
                try:
                    self.rows.append(self._sample_nvml())
                except Exception:
                    self._nvml = None
                    self.source = "nvidia-smi"
                    continue
                self._stop.wait(0.0005)
                continue
            try:
                out = subprocess.run(
                    ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                     "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5)
                if out.returncode == 0 and out.stdout.strip():
                    self.rows.append([c.strip() for c in out.stdout.strip().split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        # the timed loop is a busy Python thread: shorten the interpreter's
        # thread switch interval so the sampler gets to run while it does
        # (kernels are timed by CUDA events; the host loop only enqueues)
        self._switch = sys.getswitchinterval()
        sys.setswitchinterval(2e-4)
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        if self._t:
            self._t.join(timeout=10)
        sys.setswitchinterval(self._switch)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 2 + i and r[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(mx) if mx else None, "reasons": reasons,
                "samples": len(self.rows), "source": self.source}


def build_graph(config):
    from paper_1311_1695_b200.generators import config_graph
    return config_graph(config)


from paper_1311_1695_b200.dist import (RowPartition,  # noqa: E402
                                      device_row_ptr, local_operator,
                                      local_operator_device, partition_rows)


def cpu_spmv_threads(rp, col, val, x, nthreads, chunks):
    """Oracle SpMV (reduceat per row, sparse.py:135-139) over row chunks in
    a thread pool (numpy releases the GIL inside the ufunc loops)."""
    from concurrent.futures import ThreadPoolExecutor
    y = np.zeros(len(rp) - 1)

    def work(c):
        r0, r1 = c
        lo, hi = rp[r0], rp[r1]
        seg = val[lo:hi] * x[col[lo:hi]]
        lens = np.diff(rp[r0:r1 + 1])
        nz = np.flatnonzero(lens > 0)
        if nz.size:
            y[r0 + nz] = np.add.reduceat(seg, (rp[r0:r1] - lo)[nz])
    if nthreads == 1:
        for c in chunks:
            work(c)
    else:
        with ThreadPoolExecutor(nthreads) as ex:
            list(ex.map(work, chunks))
    return y


def bench_config(config, n, nnz, world):
    """The `config` object both arms print (identical, so the driver can pair
    the lines)."""
    return {"workload": f"{config}: one SpMV of the weighted Laplacian (BASELINE configs[3], LCC)"
                        if config == "C4" else f"{config}: one SpMV of the graph Laplacian",
            "n": n, "nnz": nnz,
            "l2": "flushed between steps (256 MiB write, untimed)",
            "parallelism": f"rows{world}" if world > 1 else "single"}


def reference_arm(args):
    """CPU reference arm: the oracle restatement of the reference SpMV."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    from oracle import lapeig_oracle as O
    g = build_graph(args.config)
    rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    n, nnz = g.n_nodes, int(rp[-1])
    x = np.random.default_rng(0).standard_normal(n)
    nthreads = os.cpu_count() or 1
    cuts = partition_rows(rp, nthreads * 4)
    chunks = [(cuts[i], cuts[i + 1]) for i in range(len(cuts) - 1)]
    y_ref = O.spmv(O.Csr(n, rp, col, val), x)
    y = cpu_spmv_threads(rp, col, val, x, nthreads, chunks)
    assert np.allclose(y, y_ref, rtol=1e-13, atol=1e-12)
    for _ in range(args.warmup):
        cpu_spmv_threads(rp, col, val, x, nthreads, chunks)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_spmv_threads(rp, col, val, x, nthreads, chunks)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * float(np.mean(times))
    value = 1e3 / ms
    algo = 12 * nnz + 8 * (n + 1) + 16 * n
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": ms, "higher_is_better": True, "scaling": "strong",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, n, nnz, int(os.environ.get("WORLD_SIZE", "1"))),
        "effective_gbs": algo / (ms * 1e-3) / 1e9,
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": nthreads, "kind": "port",
                         "sample": f"{args.steps} full {args.config} matvecs, oracle reduceat "
                                   f"SpMV row-chunked over {nthreads} threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


def cpu_baseline_sample(g, seconds=10.0):
    """Single-thread oracle SpMV (the reference's algorithm) for a bounded
    sample of ~seconds (rank 0, N = 1 only)."""
    from oracle import lapeig_oracle as O
    rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
    a = O.Csr(g.n_nodes, rp, col, val)
    x = np.random.default_rng(0).standard_normal(a.n)
    O.spmv(a, x)
    reps, t0 = 0, time.perf_counter()
    while time.perf_counter() - t0 < seconds and reps < 200:
        O.spmv(a, x)
        reps += 1
    dt = (time.perf_counter() - t0) / reps
    return {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port",
            "sample": f"{reps} oracle matvecs (np.add.reduceat, sparse.py:128-139) in "
                      f"{reps * dt:.1f} s on one host core"}


def _event_timer(fn, flush=None, reps=20):
    """Median CUDA-event time of fn() in microseconds on the current stream,
    L2 flushed before every rep (untimed) when a flush buffer is given."""
    import torch
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    s = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    e = [torch.cuda.Event(enable_timing=True) for _ in range(reps)]
    for i in range(reps):
        if flush is not None:
            flush.fill_(i & 0xff)
        s[i].record(st)
        fn()
        e[i].record(st)
    torch.cuda.synchronize()
    return 1e3 * float(np.median([a.elapsed_time(b) for a, b in zip(s, e)]))


def cpu_solvers_block(budget_s=25.0):
    """The reference solvers timed on THIS box's host cores in this run: the
    oracle's restatements of dacg_smallest / jd_smallest / irlm_smallest
    (pinned to the reference's golden eigenvalues and MVP counts,
    tests/test_oracle_golden.py), each with a shared precomputed IC(0) factor
    exactly as the reference harness does (bench.py:123-158 of the reference:
    factorisation outside the timed solve).  Runs longer than budget_s stop at
    the deadline; their wall time is projected as (time per MVP so far) x (the
    reference's MVP count), and says so.  Rank 0, N = 1 only."""
    from oracle import lapeig_oracle as O
    runs = {"C1": ("dacg", "jd", "irlm"), "C2": ("dacg", "jd"), "C3": ("jd",),
            "C4": ("dacg", "jd")}
    fns = {"dacg": O.dacg, "jd": O.jd, "irlm": O.irlm}
    out = {"cores": os.cpu_count(),
           "openblas_threads": os.environ.get("OPENBLAS_NUM_THREADS", "default"),
           "kind": "port", "note": "oracle restatement of the reference solvers; SpMV and "
           "SuperLU-equivalent triangular solves single-threaded like the reference"}
    for cfg, solvers in runs.items():
        gold = json.loads((ROOT / "tests" / "golden" / f"config_{cfg}.json").read_text())
        g = build_graph(cfg)
        rp, col, val = O.build_laplacian(g.n_nodes, g.i, g.j, g.w)
        a = O.Csr(g.n_nodes, rp, col, val)
        lrp, lcol, lval, _, _ = O.ic0_factorize(a)
        f = O.Ic0(a.n, lrp, lcol, lval)
        for name in solvers:
            r = gold["solvers"][name]
            t0 = time.perf_counter()
            rec = {"neig": gold["neig"], "delta": gold["delta"], "reference_mvp": r["mvp"]}
            try:
                res = fns[name](a, gold["neig"], delta=gold["delta"], f=f,
                                deadline=t0 + budget_s)
                rec.update(wall_s=time.perf_counter() - t0, mvp=res.mvp, projected=False,
                           eig_relerr_vs_golden=float(np.max(
                               np.abs(res.values - r["eigenvalues"]) /
                               np.abs(r["eigenvalues"]))))
            except TimeoutError:
                dt = time.perf_counter() - t0
                done = max(1, a.count)
                rec.update(wall_s=dt / done * r["mvp"], projected=True,
                           sample=f"{done} MVPs in {dt:.1f} s, projected to the reference's "
                                  f"{r['mvp']} MVPs")
            out[f"{cfg}_{name}"] = rec
    return out


def _ncu_traffic(config, world):
    """DRAM bytes (read + write) per spmv_kernel launch from the committed
    `ncu --set full` capture of this workload (profiles/), or None."""
    if world != 1:
        return None
    try:
        t = json.loads((ROOT / "profiles" / "spmv_traffic.json").read_text())
        if t.get("config") == config:
            return float(t["dram_bytes_per_launch"])
    except Exception:
        pass
    return None


def north_star_residual(a, pairs):
    """max_i ||L u_i - lambda_i u_i||_2 / ||L||_1 over the returned pairs
    (the north star's residual), next to the reference's own criterion
    ||A u - theta u|| / (||u|| |theta|) (results.py:97-104, rayleigh_residuals).
    ||L||_1 is the largest absolute column sum; L is symmetric, so the
    largest absolute row sum."""
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.results import rayleigh_residuals
    absrow = np.add.reduceat(np.abs(a.values), a.row_ptr[:-1])
    norm1 = float(absrow.max())
    U = pairs.vectors
    res = [float(np.linalg.norm(L.spmv(a, U[:, i]) - pairs.values[i] * U[:, i])) / norm1
           for i in range(U.shape[1])]
    _, ref = rayleigh_residuals(a, U)
    return {"ns_residual_max": max(res), "ref_criterion_max": float(np.max(ref)),
            "norm1_L": norm1}


def solve_block(a, f, f_mc=None):
    """Wall time to 5 eigenpairs (delta 1e-8) with DACG and JD on the device,
    with the reference's IC(0) (parity mode) and, flagged separately, with
    the multicolour-reordered IC(0) variant."""
    import torch
    import paper_1311_1695_b200 as L
    ref = {}
    try:
        ref = json.loads((ROOT / "tests/golden/config_C4.json").read_text())["solvers"]
    except Exception:
        pass
    out = {}
    runs = [("dacg", L.dacg_smallest, f, "ic0 (reference)"), ("jd", L.jd_smallest, f, "ic0 (reference)")]
    if f_mc is not None:
        runs += [("dacg_multicolor", L.dacg_smallest, f_mc, "multicolour ic0 (flagged variant)"),
                 ("jd_multicolor", L.jd_smallest, f_mc, "multicolour ic0 (flagged variant)")]
    f_fsai = L.fsai_factorize(a, kmax=32)
    f_fsai.device()
    runs += [("dacg_fsai", L.dacg_smallest, f_fsai, "fsai kmax 32 (flagged variant)"),
             ("jd_fsai", L.jd_smallest, f_fsai, "fsai kmax 32 (flagged variant)")]
    for name, fn, prec, label in runs:
        walls = []
        for _ in range(2):   # first call (graph capture, lazy scratch) and steady state
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            pairs, rep = fn(a, 5, delta=1e-8, f=prec)
            torch.cuda.synchronize()
            walls.append(time.perf_counter() - t0)
        wall = walls[1]
        r = ref.get(name.split("_")[0], {})
        err = None
        if r.get("eigenvalues"):
            err = float(np.max(np.abs(pairs.values - r["eigenvalues"]) /
                               np.abs(r["eigenvalues"])))
        out[name] = {**north_star_residual(a, pairs),
                     "wall_s": wall, "wall_s_first_call": walls[0], "mvp": rep.mvp, "neig": 5,
                     "delta": 1e-8,
                     "preconditioner": label,
                     "eig_relerr_vs_reference": err,
                     "reference_wall_s_build_container": r.get("wall_seconds"),
                     "reference_mvp": r.get("mvp")}
    return out


def solve_configs_block(prebuilt=None):
    """Wall time to k eigenpairs on the BASELINE configs with the reference's
    own solver settings (golden: neig, delta, reference IC(0)), next to the
    reference's MVPs / eigenvalues / wall time (build container): C1 DACG /
    JD / IRLM, C2 DACG / JD, C3 JD at neig 5 and at the BASELINE's 20, C4
    DACG / JD at the BASELINE's neig 10 (C4 at neig 5 is the `solve` block).
    prebuilt: {"C4": (a, f)} reuses a matrix + factor the caller holds."""
    import torch
    import paper_1311_1695_b200 as L
    runs = {"C1": ("dacg", "jd", "irlm"), "C2": ("dacg", "jd"), "C3": ("jd",),
            "C3n20": ("jd",), "C4n10": ("dacg", "jd")}
    fns = {"dacg": L.dacg_smallest, "jd": L.jd_smallest, "irlm": L.irlm_smallest}
    out = {}
    cache = dict(prebuilt or {})
    for cfg, solvers in runs.items():
        path = ROOT / "tests" / "golden" / f"config_{cfg}.json"
        if not path.exists():
            continue
        gold = json.loads(path.read_text())
        base = cfg[:2]
        if base not in cache:
            a = L.build_laplacian(L.config_graph(base))
            f = L.ic0_factorize(a)
            f.device()
            cache[base] = (a, f)
        a, f = cache[base]
        variants = [("", f, "ic0 (reference)")]
        if cfg in ("C3n20", "C4n10"):
            # the flagged FSAI variant next to the parity mode (same pairs,
            # different preconditioner: its MVPs are reported, not compared)
            ff = L.fsai_factorize(a, kmax=32)
            ff.device()
            variants.append(("_fsai", ff, "fsai kmax 32 (flagged variant)"))
            variants.append(("_ic0j3", L.ic0_jacobi_sweeps(f, 3),
                             "ic0, 3 Jacobi sweeps per triangle (flagged variant)"))
        for name in solvers:
            for suffix, prec, label in variants:
                walls = []
                for _ in range(2):
                    torch.cuda.synchronize()
                    t0 = time.perf_counter()
                    pairs, rep = fns[name](a, gold["neig"], delta=gold["delta"], f=prec)
                    torch.cuda.synchronize()
                    walls.append(time.perf_counter() - t0)
                r = gold["solvers"][name]
                ref_vals = np.asarray(r["eigenvalues"])
                out[f"{cfg}_{name}{suffix}"] = {**north_star_residual(a, pairs),
                    "neig": gold["neig"], "delta": gold["delta"], "preconditioner": label,
                    "wall_s": walls[1], "wall_s_first_call": walls[0], "mvp": rep.mvp,
                    "reference_mvp": r["mvp"],
                    "eig_relerr_vs_reference": float(np.max(np.abs(pairs.values - ref_vals)
                                                            / np.abs(ref_vals))),
                    "reference_wall_s_build_container": r["wall_seconds"],
                    "speedup_vs_reference_wall": r["wall_seconds"] / walls[1]}
    return out


class _OverlappedProduct:
    """One rank's product of the row-partitioned SpMV with the exchange
    overlapped: interior half (own columns + diagonal) while the NCCL slice
    exchange runs, exterior half accumulated after it (lg_csr_split_cols /
    lg_spmv_acc); the plain exchange-then-product when the block is not
    packed."""

    def __init__(self, dist, part, rank, op):
        from paper_1311_1695_b200.dist import RowComm, TorchBackend, split_cols
        self.comm = RowComm(part, rank, TorchBackend(dist))
        self.op = op
        self.halves = split_cols(op, *part.rows(rank)) if op.packed else None

    def __call__(self, x, y):
        from paper_1311_1695_b200._plan import SpmvAcc
        if self.halves is None:
            self.comm.exchange_(x)
            self.op.matvec(x, y)
            return
        inner, outer = self.halves
        reqs = self.comm.exchange_start(x)
        inner.matvec(x, y)
        self.comm.exchange_wait(reqs)
        SpmvAcc(outer, x, y)()


def solve_dist_block(a, dist=None, world=1, rank=0, neig=10, delta=1e-8):
    """Row-partitioned DACG and JD on C4 at the BASELINE's neig 10, delta
    1e-8: every rank owns a row block and its slice of every
    solver vector; one all-reduce per dot pass, one slice exchange per SpMV
    (overlapped with the interior product).  Preconditioner: FSAI (flagged
    variant; two row-partitioned SpMVs), the same operator at every N, so
    the MVP counts do not depend on N (the reference's natural-order IC(0)
    does not shard).  Time to solution = max over ranks (factorization
    excluded, as in the reference harness bench.py:123-125)."""
    import torch
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200.dist import (SOLVER_ROW_WEIGHT, RowComm, RowPartition,
                                           TorchBackend)
    part = RowPartition(a.row_ptr, world, SOLVER_ROW_WEIGHT)
    comm = RowComm(part, rank, TorchBackend(dist) if dist else None)
    f = L.fsai_factorize(a, kmax=32)
    f.device()
    try:
        gj = json.loads((ROOT / "tests/golden/config_C4n10.json").read_text())
        gold = gj["solvers"] if (gj.get("n") == a.n and gj.get("neig") == neig) else {}
    except Exception:
        gold = {}
    out = {}
    for name, fn in (("dacg", L.dacg_smallest), ("jd", L.jd_smallest)):
        walls = []
        for _ in range(2):   # first call and steady state
            torch.cuda.synchronize()
            if dist:
                dist.barrier()
            t0 = time.perf_counter()
            pairs, rep = fn(a, neig, delta=delta, f=f, comm=comm)
            torch.cuda.synchronize()
            w = time.perf_counter() - t0
            if dist:
                t = torch.tensor([w], device="cuda", dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                w = float(t.item())
            walls.append(w)
        r = {"neig": neig, "delta": delta, "n_gpus": world, "wall_s": walls[1],
             "wall_s_first_call": walls[0], "mvp": rep.mvp,
             "preconditioner": "fsai kmax 32 (flagged; the same at every N)",
             "parallelism": f"rows{world}" if world > 1 else "single"}
        g = gold.get(name)
        if g:
            ref = np.asarray(g["eigenvalues"])
            r["eig_relerr_vs_reference"] = float(np.max(np.abs(pairs.values - ref) / ref))
            r["reference_mvp"] = g["mvp"]
            r["reference_wall_s_build_container"] = g["wall_seconds"]
        out[name] = r
    return out


def c5_block(peaks, steps=10, dist=None, world=1, rank=0, solve=True):
    """BASELINE configs[4] (R-MAT scale 26, edge factor 16, ~2.1e9 nonzeros):
    device-side ingest (sampling, dedupe, largest component, packed
    Laplacian) and the SpMV on it -- at N > 1 row-partitioned by nonzeros
    (each rank builds the same graph, keeps its row block in the padded
    block, every rank's slice of x exchanged in place per product with one
    NCCL point-to-point group; time = max over ranks).  Not buildable by the reference; reported next to
    the headline, not as it."""
    import torch
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = rmat_laplacian_device(26, 16, seed=0)
    torch.cuda.synchronize()
    build = time.perf_counter() - t0
    n = A.n
    xh = np.random.default_rng(0).standard_normal(n)
    gather = None
    x = dev.to_device(xh)
    y = dev.empty(n)
    if world > 1:
        part = RowPartition(device_row_ptr(A.device()), world)
        d = local_operator_device(A.device(), part, rank)
        A._dev = None          # the full matrix is no longer needed on this rank
        torch.cuda.empty_cache()
        gather = _OverlappedProduct(dist, part, rank, d)
    else:
        d = A.device()

    def step():
        if gather is not None:
            gather(x, y)
        else:
            d.matvec(x, y)

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
    for i in range(steps):
        e0[i].record()
        step()
        e1[i].record()
    torch.cuda.synchronize()
    ms = float(np.mean([p.elapsed_time(q) for p, q in zip(e0, e1)]))
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    out = {"workload": "C5: R-MAT scale 26 ef 16 (a,b,c)=(.57,.19,.19), LCC, unit weights, "
                       "device-built (counter-based RNG)",
           "n": n, "m": A.m, "nnz": A.nnz, "n_gpus": world,
           "parallelism": f"rows{world} (nnz-balanced row blocks, in-place P2P exchange "
                          "of x per product)" if world > 1 else "single",
           "build_s": build, "spmv_ms": ms, "matvecs_per_s": 1e3 / ms,
           "stream_gbs_rank0": d.stream_bytes / (ms * 1e-3) / 1e9,
           "effective_gbs": (12 * A.nnz + 8 * (n + 1) + 16 * n) / (ms * 1e-3) / 1e9,
           "frac_stream_of_hbm_rank0": d.stream_bytes / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
           "l2": "x (262 MB) exceeds L2; not flushed"}
    if world == 1 and solve:
        # BASELINE configs[4]'s solve: 5 smallest pairs by DACG at delta 1e-8
        # (flagged FSAI built on the device; the reference cannot build C5),
        # certified by fresh residuals
        import paper_1311_1695_b200 as L
        from paper_1311_1695_b200.precond import FsaiFactor
        from paper_1311_1695_b200.results import rayleigh_residuals
        del x, y
        torch.cuda.empty_cache()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        f = FsaiFactor.from_device(A, kmax=32)
        torch.cuda.synchronize()
        setup = time.perf_counter() - t0
        t0 = time.perf_counter()
        pairs, rep = L.dacg_smallest(A, 5, delta=1e-8, f=f)
        torch.cuda.synchronize()
        wall = time.perf_counter() - t0
        _, res = rayleigh_residuals(A, pairs.vectors)
        out["solve"] = {"solver": "dacg", "neig": 5, "delta": 1e-8, "wall_s": wall,
                        "mvp": rep.mvp, "preconditioner": "fsai kmax 32, device setup (flagged)",
                        "preconditioner_setup_s": setup,
                        "eigenvalues": [float(v) for v in pairs.values],
                        "max_fresh_residual": float(np.max(res)),
                        "residuals_within_delta": bool(np.max(res) <= 1e-8)}
        del f, pairs
        x = y = None
    del A, d, x, y
    torch.cuda.empty_cache()
    return out


def c5_main(args):
    """`--config C5`: BASELINE configs[4] as a first-class bench line -- the
    largest single-GPU configuration (R-MAT scale 26, 2.14e9 nonzeros,
    device-built; the reference cannot build it).  A step is one matvec of
    the panelled product; x (262 MB) exceeds L2, so nothing is flushed.  At
    N > 1 each rank multiplies its nnz-balanced row block after the in-place
    slice exchange (time = max over ranks)."""
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev
    from paper_1311_1695_b200.device_graphs import rmat_laplacian_device
    peaks, peak_kind = _peaks()
    A = rmat_laplacian_device(26, 16, seed=0, panels=(world == 1))
    n = A.n
    xh = np.random.default_rng(0).standard_normal(n)
    x, y = dev.to_device(xh), dev.empty(n)
    gather = None
    if world > 1:
        part = RowPartition(device_row_ptr(A.device()), world)
        d = local_operator_device(A.device(), part, rank)
        gather = _OverlappedProduct(dist, part, rank, d)
    else:
        d = A.device()

    def step():
        if gather is not None:
            gather(x, y)
        else:
            d.matvec(x, y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    st = torch.cuda.current_stream()
    e0 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    e1 = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            e0[i].record(st)
            step()
            e1[i].record(st)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    ms = float(np.mean([p.elapsed_time(q) for p, q in zip(e0, e1)]))
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    algo = 12 * A.nnz + 8 * (n + 1) + 16 * n
    stream = d.stream_bytes
    # x gathers of the whole stored column stream alone (one pass, no panels)
    gather_us = _event_timer(lambda: d.gather_probe(x), reps=5) if world == 1 else None
    traffic = None
    try:
        tr = json.loads((ROOT / "profiles" / "spmv_traffic_c5.json").read_text())
        traffic = float(tr["dram_bytes_per_product"]) if world == 1 else None
    except Exception:
        pass
    launches_per_step = (1 + 2 * getattr(d, "npanels", 0)) if world == 1 and getattr(
        d, "npanels", 0) > 1 else 2
    line = {
        "metric": METRIC, "value": 1e3 / ms, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic (device-built R-MAT, counter-based RNG)",
        "config": {"workload": "C5: one SpMV of the R-MAT scale 26 ef 16 Laplacian (BASELINE "
                               "configs[4], LCC, unit weights)", "n": n, "nnz": A.nnz,
                   "l2": "x (262 MB) and the 8.5 GB stream exceed L2; not flushed",
                   "parallelism": f"rows{world}" if world > 1 else "single"},
        "effective_gbs": algo / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": stream / (ms * 1e-3) / 1e9,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": stream / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                     "traffic": traffic, "peak_kind": peak_kind, "bytes_per_launch": stream,
                     "format": "packed Laplacian, 4 column panels (x slices L2-resident)"
                               if world == 1 else "packed row block",
                     "bytes_model": "diag init 24 n + per panel: 4 B / off-diagonal + 96 B / "
                                    "warp block + 8 B / column of its x slice + 20 B / row "
                                    "written (y read-modify-write, row map)",
                     "gather_floor_us": gather_us,
                     "frac_of_gather_floor": gather_us / (ms * 1e3) if gather_us else None,
                     "gather_gsectors_s": (A.nnz - n) / (gather_us * 1e-6) / 1e9
                     if gather_us else None},
        "gpu_launches": args.steps * launches_per_step,
        "clocks": clk.summary(),
    }
    if rank == 0:
        reps = 3
        L.spmv(A, xh)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            L.spmv(A, xh)
        line["e2e"] = {"value": reps / (time.perf_counter() - t0), "unit": UNIT,
                       "h2d_bytes_per_step": 8 * n, "d2h_bytes_per_step": 8 * n,
                       "path": "paper_1311_1695_b200.spmv(A, numpy x) -> numpy y"}
    if rank == 0 and world == 1 and not args.no_cpu:
        # the reference's SpMV on a bounded sample: the host CSR (exported
        # from the device, bit-exact) restricted to the first 1/64 of the
        # nonzeros, one host core, scaled to a whole matvec
        from oracle import lapeig_oracle as O
        from paper_1311_1695_b200 import _native as nat
        rp = np.empty(n + 1, dtype=np.int64)
        col = np.empty(A.nnz, dtype=np.int64)
        val = np.empty(A.nnz)
        nat.call("lg_csr_export_host", d.handle, rp.ctypes.data, col.ctypes.data, val.ctypes.data)
        r1 = int(np.searchsorted(rp, A.nnz // 64))
        sub = O.Csr(r1, rp[:r1 + 1].copy(), col[:rp[r1]], val[:rp[r1]])
        sub.n = n   # columns index all of x
        O.spmv(sub, xh)
        t0 = time.perf_counter()
        O.spmv(sub, xh)
        dt = (time.perf_counter() - t0) * A.nnz / max(1, int(rp[r1]))
        line["cpu_baseline"] = {"value": 1.0 / dt, "unit": UNIT, "cores": 1, "kind": "port",
                                "sample": f"oracle reduceat SpMV over the first {r1} rows "
                                          f"({int(rp[r1])} nonzeros, 1/64 of the matrix), "
                                          "one host core, scaled to a whole matvec"}
        del rp, col, val, sub
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser(description=__doc__, formatter_class=argparse.RawTextHelpFormatter)
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=50)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="b200", choices=("b200", "reference"))
    ap.add_argument("--config", default="C4")
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-c5", action="store_true")
    ap.add_argument("--no-vendor", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return reference_arm(args)
    if args.config == "C5":
        return c5_main(args)

    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only knobs: LG_BENCH_BACKEND=gloo with LG_BENCH_SAME_GPU=1 runs the
    # N > 1 code with every rank on cuda:0 (two processes sharing one GPU)
    if os.environ.get("LG_BENCH_SAME_GPU") == "1":
        local = 0
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        backend = os.environ.get("LG_BENCH_BACKEND", "nccl")
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        else:
            dist.init_process_group(backend)

    import paper_1311_1695_b200 as L
    from paper_1311_1695_b200 import _device as dev

    g = build_graph(args.config)
    a = L.build_laplacian(g)
    n, nnz = a.n, a.nnz
    part = RowPartition(a.row_ptr, world)
    cuts = part.cuts
    r0, r1 = cuts[rank], cuts[rank + 1]
    xh0 = np.random.default_rng(0).standard_normal(n)
    x = dev.to_device(xh0)
    y = dev.empty(n)
    gather = None
    if world == 1:
        d = a.device()
    else:
        # this rank's rows (global columns); the exchange moves every rank's
        # slice of x to every peer in place (one NCCL P2P group per product)
        d = local_operator(a, part, rank)
        gather = _OverlappedProduct(dist, part, rank, d)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream()

    def step():
        if gather is not None:
            # every rank owns rows r0..r1 of the iterate; the interior
            # product runs while the slices of x are exchanged, the exterior
            # product accumulates after the exchange
            gather(x, y)
        else:
            d.matvec(x, y)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        for i in range(args.steps):
            flush.fill_(i & 0xff)            # evict L2 between steps (not timed)
            starts[i].record(stream)
            step()
            ends[i].record(stream)
        torch.cuda.synchronize()
    if dist:
        dist.barrier()
    step_ms = [s.elapsed_time(e) for s, e in zip(starts, ends)]
    ms = float(np.mean(step_ms))
    if dist:
        t = torch.tensor([ms], device="cuda", dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    value = 1e3 / ms
    algo = 12 * nnz + 8 * (n + 1) + 16 * n
    # kernel-only roofline (the SpMV launch of this rank): the bytes the
    # stored format actually streams (packed Laplacian words when eligible)
    local_nnz = int(a.row_ptr[r1] - a.row_ptr[r0])
    local_rows = r1 - r0
    local_algo = 12 * local_nnz + 8 * (local_rows + 1) + 16 * local_rows + 8 * (n - local_rows)
    if d.packed:
        local_stream = 4 * (local_nnz - local_rows) + 8 * (local_rows + 1) + 8 * local_rows \
            + 16 * local_rows + 8 * (n - local_rows)
    else:
        local_stream = local_algo
    if world == 1:
        local_stream = d.stream_bytes   # exactly what the launch streams (lg_csr_info)
    peaks, peak_kind = _peaks()
    # e2e through the public API with host buffers (rank 0 replica path)
    xh = np.random.default_rng(1).standard_normal(n)
    e2e = None
    if rank == 0:
        for _ in range(3):
            L.spmv(a, xh)
        torch.cuda.synchronize()
        reps = max(5, min(args.steps, 30))
        t0 = time.perf_counter()
        for _ in range(reps):
            L.spmv(a, xh)
        e2e_s = (time.perf_counter() - t0) / reps
        e2e = {"value": 1.0 / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * n,
               "d2h_bytes_per_step": 8 * n,
               "path": "paper_1311_1695_b200.spmv(a, numpy x) -> numpy y"
                       + (" (rank 0, whole matrix)" if world > 1 else "")}
        # the same through the C ABI a reference-side binding would call
        # (lg_spmv_host: host x in, host y out)
        import ctypes
        from paper_1311_1695_b200 import _native as nat
        yh = np.empty(n)
        xd_, yd_ = dev.empty(n), dev.empty(n)
        args_c = (a.device().handle, xh.ctypes.data, yh.ctypes.data,
                  ctypes.c_void_p(xd_.data_ptr()), ctypes.c_void_p(yd_.data_ptr()),
                  ctypes.c_void_p(torch.cuda.current_stream().cuda_stream))
        for _ in range(3):
            nat.call("lg_spmv_host", *args_c)
        t0 = time.perf_counter()
        for _ in range(reps):
            nat.call("lg_spmv_host", *args_c)
        e2e["cabi_value"] = reps / (time.perf_counter() - t0)
        e2e["cabi_path"] = "lg_spmv_host(csr, x_h, y_h, ...) (C ABI, pinned staging)"
    # the product's real bound: its x gathers alone (lg_spmv_gather_probe: the
    # stored column stream, eight gathers in flight per thread, nothing
    # else), timed live on this operator under the same L2 flush
    gather_us = _event_timer(lambda: d.gather_probe(x), flush=flush, reps=10)
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": bench_config(args.config, n, nnz, world),
        "effective_gbs": algo / (ms * 1e-3) / 1e9,
        "roofline": {"bound": "hbm", "achieved": local_stream / (ms * 1e-3) / 1e9,
                     "peak": peaks["hbm_gbs"], "unit": "GB/s",
                     "frac": local_stream / (ms * 1e-3) / 1e9 / peaks["hbm_gbs"],
                     "traffic": _ncu_traffic(args.config, world), "peak_kind": peak_kind,
                     "bytes_per_launch": local_stream,
                     "format": "packed Laplacian (4 B / off-diagonal + diag vector)"
                               if d.packed else "CSR f64 / int32",
                     "bytes_model": ("4 (nnz - n) + 96 B per warp block (row structure) + 8 n "
                                     "(diagonal) + 16 n (x, y) (packed)" if d.packed
                                     else "12 nnz + 96 B per warp block + 16 n"),
                     "effective_bytes_model": "12 nnz + 8 (n+1) + 16 n (SURVEY 8(d))",
                     # the kernel is bound by the rate at which the SMs get
                     # random 32-byte sectors of x out of L2 (one gather per
                     # stored off-diagonal: ~230 G sectors/s on this part,
                     # whatever the grid, cache operator, lane mapping or a
                     # shared-memory table of the hub columns),
                     # not by HBM: gather_floor_us is that gather stream
                     # alone, timed live on this operator
                     "gather_floor_us": gather_us,
                     "frac_of_gather_floor": gather_us / (ms * 1e3),
                     "gather_gsectors_s": (local_nnz - local_rows) / (gather_us * 1e-6) / 1e9},
        "gpu_launches": args.steps,
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    line_factor = {}
    if rank == 0 and world == 1 and not args.no_solve:
        f = L.ic0_factorize(a)
        line_factor["f"] = f
        f_mc = L.ic0_factorize_multicolor(a)
        f.device()
        f_mc.device()   # device factor upload = setup, like the reference's splu
        line["solve"] = solve_block(a, f, f_mc)
        line["solve_configs"] = solve_configs_block({"C4": (a, f)})
    if not args.no_solve and args.config == "C4":
        sd = solve_dist_block(a, dist=dist, world=world, rank=rank)
        if rank == 0:
            line["solve_dist"] = sd
    if not args.no_c5:
        c5 = c5_block(peaks, dist=dist, world=world, rank=rank, solve=not args.no_solve)
        if rank == 0:
            line["c5"] = c5
    if rank == 0 and world == 1 and not args.no_cpu:
        line["cpu_baseline"] = cpu_baseline_sample(g)
        if not args.no_solve:
            cs = cpu_solvers_block()
            line["cpu_solvers"] = cs
            # time-to-solution speed-up against the reference solvers timed on
            # this box in this run (same graph, neig, delta, preconditioner)
            for blk, key_of in (("solve_configs", lambda k: k),
                                ("solve", lambda k: "C4_" + k)):
                for k, v in line.get(blk, {}).items():
                    if "preconditioner" in v and "reference" not in v["preconditioner"]:
                        base = k.rsplit("_", 1)[0] if blk == "solve_configs" else k.split("_")[0]
                    else:
                        base = k
                    c = cs.get(key_of(base))
                    if c and v.get("wall_s"):
                        v["reference_wall_s_same_box"] = c["wall_s"]
                        v["reference_wall_projected"] = c["projected"]
                        v["speedup_vs_reference_same_box"] = c["wall_s"] / v["wall_s"]
    if rank == 0 and world == 1 and not args.no_vendor:
        sys.path.insert(0, str(ROOT / "scripts"))
        from vendor_cusparse import vendor_block
        fv = line_factor.get("f")
        line["vendor"] = vendor_block(a, fv, x, _event_timer, flush)
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
