"""Shared fixtures.  GPU tests are marked ``@pytest.mark.gpu``; everything
else runs on a CPU-only host.  ``oracle/`` (the CPU checker) is imported only
from tests, smoke() and bench.py."""

import glob
import os
import sys

import numpy as np
import pytest

REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, REPO)
GOLDEN = os.path.join(REPO, "tests", "golden")


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200)")


def golden_cases():
    return sorted(glob.glob(os.path.join(GOLDEN, "case_*.npz")))


def load_case(path):
    z = np.load(path, allow_pickle=False)
    d = {k: z[k] for k in z.files}
    for k in ("n_rows", "n_cols", "C", "sigma", "align_bytes", "n_rows_padded",
              "n_chunks"):
        d[k] = int(d[k])
    d["permute_cols"] = bool(d["permute_cols"])
    d["name"] = str(d["name"])
    return d


def case_id(path):
    return os.path.basename(path)[5:-4]


@pytest.fixture
def rng():
    return np.random.default_rng(20240901)


def random_crs(rng, n_rows, n_cols, nnz_target, allow_zero_values=False):
    """Seeded random canonical CRS (the reference fixture's recipe,
    pkg/tests/conftest.py:10-27)."""
    from paper_1307_6209_b200 import COOMatrix, coo_to_crs
    nnz_target = min(nnz_target, n_rows * n_cols)
    if nnz_target <= 0:
        return coo_to_crs(COOMatrix(n_rows, n_cols, np.empty(0, np.int32),
                                    np.empty(0, np.int32), np.empty(0)))
    flat = rng.choice(n_rows * n_cols, size=nnz_target, replace=False)
    vals = rng.uniform(-1.0, 1.0, size=nnz_target)
    if allow_zero_values:
        vals[rng.random(nnz_target) < 0.05] = 0.0
    return coo_to_crs(COOMatrix(n_rows, n_cols, flat // n_cols, flat % n_cols, vals))


def dense_of(m):
    d = np.zeros((m.n_rows, m.n_cols))
    rows = np.repeat(np.arange(m.n_rows), np.diff(m.rpt))
    np.add.at(d, (rows, m.col), m.val)
    return d
