"""The reference's own test suite (pkg/tests/*.py), restated case by case,
run against this package under the reference's module name.

`lapeig` below IS paper_1311_1695_b200 (every submodule the reference tests
import is aliased), so each test reads like the reference test it restates:
same fixture graphs (the package's restatement of the reference generators,
pinned bit-exact in tests/test_oracle_golden.py), same inputs, same known
answers, same tolerances.  Each test cites the reference case it restates.
The shared oracles of the reference conftest (pkg/tests/conftest.py:10-31)
are restated here.
"""

import importlib
import sys

import numpy as np
import pytest

import paper_1311_1695_b200 as _pkg

sys.modules["lapeig"] = _pkg
for _sub in ("dacg", "generators", "graphs", "ic0", "irlm", "jd", "kernels", "pcg",
             "results", "sparse", "spectral"):
    sys.modules[f"lapeig.{_sub}"] = importlib.import_module(f"paper_1311_1695_b200.{_sub}")


def dense_positive_pairs(edges, neig=None):
    """Dense eigh of the Laplacian, kernel dropped at 1e-9 (conftest.py:10-23)."""
    from lapeig.graphs import build_laplacian
    from lapeig.results import EigenPairSet
    lap = build_laplacian(edges)
    w, v = np.linalg.eigh(lap.toarray())
    keep = w > 1e-9
    w, v = w[keep][:neig], v[:, keep][:, :neig]
    return EigenPairSet(values=w, vectors=v, residuals=np.zeros(w.size)), lap


def random_spd(n, rng, density=0.3):
    """B B^T + n I with B a sparsified Gaussian (conftest.py:26-31)."""
    b = rng.standard_normal((n, n))
    b[rng.random((n, n)) > density] = 0.0
    return b @ b.T + n * np.eye(n)


@pytest.fixture
def rng():
    return np.random.default_rng(12345)
