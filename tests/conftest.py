"""Shared fixtures.  `gpu` marks tests that need a CUDA device (B200)."""

import json
import sys
from pathlib import Path

import numpy as np
import pytest

ROOT = Path(__file__).resolve().parent.parent
GOLDEN = ROOT / "tests" / "golden"
if str(ROOT) not in sys.path:
    sys.path.insert(0, str(ROOT))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (sm_100a)")
    config.addinivalue_line("markers", "slow: larger BASELINE configurations")


@pytest.fixture(scope="session")
def kat():
    """Golden fixture graphs and the reference's results on them."""
    graphs = np.load(GOLDEN / "kat_graphs.npz")
    arrays = np.load(GOLDEN / "kat_arrays.npz")
    results = json.loads((GOLDEN / "kat_results.json").read_text())["graphs"]
    return graphs, arrays, results


def kat_edges(graphs, name):
    n = int(graphs[name + "_n"][0])
    return n, graphs[name + "_i"], graphs[name + "_j"], graphs[name + "_w"]


def golden_config(name):
    return json.loads((GOLDEN / f"config_{name}.json").read_text())


@pytest.fixture
def rng():
    return np.random.default_rng(12345)


def cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False
