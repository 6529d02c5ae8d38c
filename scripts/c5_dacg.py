"""BASELINE configs[4] eigen-solve: the 5 smallest nonzero eigenpairs of the
R-MAT scale-26 Laplacian (device-built, LCC, unit weights) by DACG at
delta = 1e-8, on one GPU.

The reference cannot build or factor this matrix, so the
preconditioner is the flagged Jacobi variant (the diagonal of a device-only
matrix; host IC(0) would need the matrix on the host), and parity is
residual-certified: every returned pair is re-verified with fresh products
(rayleigh_residuals, results.py:90-105), orthonormality and orthogonality to
the constant kernel vector are measured, and the smallest pairs are
cross-checked against JD when --jd is given.

usage: python scripts/c5_dacg.py [scale=26] [edge_factor=16] [neig=5] [--jd] [--fsai]
Prints one JSON line (profiles/ keeps the round's copy).
"""
import json
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1311_1695_b200 as L  # noqa: E402
from paper_1311_1695_b200 import _device as dev  # noqa: E402
from paper_1311_1695_b200.device_graphs import rmat_laplacian_device  # noqa: E402
from paper_1311_1695_b200.precond import JacobiFactor  # noqa: E402
from paper_1311_1695_b200.results import rayleigh_residuals  # noqa: E402


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    scale = int(args[0]) if len(args) > 0 else 26
    ef = int(args[1]) if len(args) > 1 else 16
    neig = int(args[2]) if len(args) > 2 else 5
    delta = 1e-8
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A = rmat_laplacian_device(scale, ef, seed=0)
    torch.cuda.synchronize()
    t_build = time.perf_counter() - t0
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if "--fsai" in sys.argv:
        from paper_1311_1695_b200.precond import FsaiFactor
        f = FsaiFactor.from_device(A, kmax=32)
        label = "fsai kmax 32, device setup (flagged; reference IC(0) infeasible)"
    else:
        f = JacobiFactor(A)
        label = "jacobi (flagged; reference IC(0) infeasible)"
    torch.cuda.synchronize()
    t_setup = time.perf_counter() - t0
    out = {"workload": f"R-MAT scale {scale} ef {ef} (a,b,c)=(.57,.19,.19), LCC, unit weights, "
                       "device-built", "n": A.n, "m": A.m, "nnz": A.nnz, "neig": neig,
           "delta": delta, "preconditioner": label, "build_s": t_build,
           "preconditioner_setup_s": t_setup}
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    pairs, rep = L.dacg_smallest(A, neig, delta=delta, f=f, seed=0)
    torch.cuda.synchronize()
    out["dacg"] = {"wall_s": time.perf_counter() - t0, "mvp": rep.mvp,
                   "iterations": rep.inner_its_total, "eigenvalues": list(map(float, pairs.values)),
                   "residuals_reported": list(map(float, rep.per_pair_residuals)),
                   "iterations_per_pair": rep.config.get("iterations_per_pair")}
    v = dev.to_device(np.ascontiguousarray(pairs.vectors))
    th, res = rayleigh_residuals(A, v)
    vt = torch.as_tensor(v)
    gram = (vt.T @ vt).cpu().numpy()
    e = torch.full((A.n,), 1.0 / np.sqrt(A.n), dtype=torch.float64, device="cuda")
    out["dacg"]["verify"] = {
        "rayleigh": list(map(float, th)), "residuals_fresh": list(map(float, res)),
        "max_residual_le_delta": bool(np.max(res) <= delta),
        "orthonormality": float(np.max(np.abs(gram - np.eye(neig)))),
        "kernel_overlap": float(torch.max(torch.abs(e @ vt)).item())}
    if "--jd" in sys.argv:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        p2, r2 = L.jd_smallest(A, neig, delta=delta, f=f, seed=0)
        torch.cuda.synchronize()
        out["jd"] = {"wall_s": time.perf_counter() - t0, "mvp": r2.mvp,
                     "eigenvalues": list(map(float, p2.values))}
        out["dacg_vs_jd_max_relerr"] = float(np.max(np.abs(pairs.values - p2.values) / p2.values))
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
