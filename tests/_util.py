import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")


def random_csc(rng, N, max_deg, allow_zero=True):
    """Uniformly random small CSC (independent of the R-MAT recipe) for brute-force pins."""
    lo = 0 if allow_zero else 1
    deg = rng.integers(lo, max_deg + 1, size=N)
    indptr = np.zeros(N + 1, np.int64)
    indptr[1:] = np.cumsum(deg)
    indices = rng.integers(0, N, size=int(indptr[-1])).astype(np.int32)
    return indptr, indices
