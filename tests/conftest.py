import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "oracle"))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) and the built CUDA library")
    config.addinivalue_line("markers", "slow: long-running CPU cross-check")


def load_golden(name):
    return np.load(os.path.join(GOLDEN, name + ".npz"))


@pytest.fixture(scope="session")
def co():
    from oracle import COracle
    return COracle()


@pytest.fixture(scope="session")
def ro():
    from oracle import ref_oracle
    r = ref_oracle()
    if r is None:
        pytest.skip("oracle/_ref (reference compiled in place) not built here")
    return r


def _cuda_ok():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


@pytest.fixture(scope="session")
def zen():
    """The product library; on a GPU box a missing build is a failure, not a skip."""
    if not _cuda_ok():
        pytest.skip("no CUDA device")
    import paper_2309_13254_b200 as z
    return z
