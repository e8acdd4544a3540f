import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: long-running full-size parity case")


def rel_diff(a, b):
    """tests/helpers.hpp:21-27: ||a - b||_F / ||b||_F (b the reference)."""
    import numpy as np
    nb = np.linalg.norm(b)
    return float(np.linalg.norm(a - b) / (nb if nb else 1.0))


@pytest.fixture(scope="session")
def ref():
    import oracle.ref as R
    if not R.available():
        pytest.skip("oracle/_ref not built (make -C oracle)")
    return R


@pytest.fixture(scope="session")
def gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_1905_09539_b200 as T
    return T
