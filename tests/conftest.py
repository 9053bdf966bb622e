import os
import sys

import numpy as np
import pytest

ROOT = os.path.abspath(os.path.join(os.path.dirname(__file__), ".."))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200) and libgdiff.so")


def load_golden(name):
    return dict(np.load(os.path.join(GOLDEN, name), allow_pickle=False))


def golden_graph(d, name):
    from paper_2410_21634_b200.graph import CsrGraph
    return CsrGraph(n=int(d[f"graph/{name}/n"]), offsets=d[f"graph/{name}/offsets"],
                    targets=d[f"graph/{name}/targets"])


@pytest.fixture(scope="session")
def small():
    return load_golden("small.npz")


@pytest.fixture(scope="session")
def pa():
    return load_golden("pa2000.npz")


@pytest.fixture(scope="session")
def cora():
    return load_golden("cora.npz")


@pytest.fixture(scope="session")
def dyn():
    return load_golden("dynamic.npz")


@pytest.fixture(scope="session")
def glob():
    return load_golden("global.npz")


@pytest.fixture(scope="session")
def gpu():
    """Skip-free guard: GPU tests must run on a GPU box and load the library."""
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2410_21634_b200 import _lib
    from paper_2410_21634_b200.build import build
    build()
    return _lib.load()
