import os
import sys

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)
GOLDEN = os.path.join(ROOT, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (CUDA path through the C-ABI)")
    config.addinivalue_line("markers", "slow: longer CPU test")


@pytest.fixture(scope="session")
def tiny_graph():
    """Small symmetrised R-MAT (synth recipe), CPU arrays."""
    import synth
    indptr, indices = synth.rmat_csc(2000, 20000, seed=11)
    return indptr.numpy(), indices.numpy()

