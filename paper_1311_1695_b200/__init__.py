"""B200-native hot path of lapeig (arXiv 1311.1695): smallest eigenpairs of
graph Laplacians by DACG, Jacobi-Davidson and inverse Lanczos, with the
shared inner loop (CSR SpMV, IC(0) apply, deflation projections, Rayleigh
quotient dots, Gram-Schmidt, JD's projected correction operator) running as
hand-written sm_100a CUDA kernels behind a C ABI (include/lapb200.h).

The public names mirror the reference package's (lapeig/__init__.py) for the
hot path, so `import paper_1311_1695_b200 as lapeig` drops in for it.
Everything that computes requires a CUDA device: there is no CPU fallback.
"""

from .dacg import dacg_smallest
from .generators import (
    ba_graph,
    chung_lu_graph,
    complete_graph,
    config_graph,
    cycle_graph,
    geometric_graph,
    grid_graph,
    path_graph,
    random_connected_graph,
    rmat_graph,
    star_graph,
)
from .graphs import (EdgeList, GraphFormatError, GraphStats, build_laplacian,
                     connected_components, csr_connected_components, largest_component,
                     load_edge_list, stats, write_matrix_market)
from .ic0 import (
    Ic0Error,
    Ic0Factor,
    MulticolorIc0Factor,
    ic0_factorize,
    ic0_factorize_multicolor,
    identity_factor,
)
from .irlm import irlm_smallest, ncv_for
from .jd import jd_smallest
from .kernels import GramSchmidtBreakdown, dense_sym_eig, mgs_orthonormalize, tridiag_eig
from .pcg import DeflationBasis, PcgOutcome, jd_correction_solve, kernel_basis, pcg_solve
from .precond import (FsaiFactor, Ic0JacobiFactor, JacobiFactor, fsai_factorize,
                      ic0_jacobi_sweeps)
from .results import EigenPairSet, SolverError, SolverReport, rayleigh_residuals
from .sparse import CsrMatrix, MvpCounter, spmv
from . import spectral
from .spectral import (PinvApprox, cut_weight, estimate_lambda_max, fiedler, fiedler_order,
                       gap_ratios, make_pinv, partition_relaxed, pinv_apply, pinv_dense,
                       sign_partition)

__version__ = "0.1.0"

__all__ = [
    "CsrMatrix", "DeflationBasis", "EdgeList", "EigenPairSet", "GramSchmidtBreakdown",
    "FsaiFactor", "fsai_factorize", "Ic0JacobiFactor", "ic0_jacobi_sweeps", "GraphFormatError", "GraphStats", "load_edge_list",
    "stats", "csr_connected_components", "write_matrix_market", "Ic0Error", "Ic0Factor", "JacobiFactor", "MulticolorIc0Factor", "ic0_factorize_multicolor", "MvpCounter", "PcgOutcome", "SolverError",
    "SolverReport", "ba_graph", "build_laplacian", "chung_lu_graph", "complete_graph",
    "config_graph", "connected_components", "cycle_graph", "dacg_smallest", "dense_sym_eig",
    "grid_graph", "ic0_factorize", "identity_factor", "irlm_smallest", "jd_correction_solve",
    "jd_smallest", "kernel_basis", "largest_component", "mgs_orthonormalize", "ncv_for",
    "path_graph", "pcg_solve", "rayleigh_residuals", "rmat_graph", "spmv", "star_graph",
    "tridiag_eig", "spectral", "PinvApprox", "cut_weight", "estimate_lambda_max", "fiedler",
    "fiedler_order", "gap_ratios", "make_pinv", "partition_relaxed", "pinv_apply", "pinv_dense",
    "sign_partition", "geometric_graph", "random_connected_graph",
]
