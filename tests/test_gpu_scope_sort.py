"""The device sigma-window sort (csrc/sellb_build.cu k_scope_sort: one CTA
per window of <= 4096 rows, block radix sort over the length bits only,
order / perm / row_lengths / chunk widths in one launch) and the wide-scope
path (device radix sort) against the oracle's restatement of
formats.py:285-393 -- heavy length ties (the index tie-break), a partial
last window, every CTA shape, empty rows, lengths needing many key bits."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix

pytestmark = pytest.mark.gpu
ARRAYS = ("cs", "cl", "col", "val", "perm", "row_lengths")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def tie_heavy(n, n_cols, seed, long_max=9):
    """Row lengths from a tiny alphabet (so most rows tie), a few long ones."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, long_max, n)
    lens[rng.random(n) < 0.001] = rng.integers(300, 5000)
    lens = np.minimum(lens, n_cols)
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, k, replace=False)) for k in lens]
                         + [np.zeros(0, np.int64)]).astype(np.int32)
    val = rng.uniform(-1, 1, int(rpt[-1]))
    return CRSMatrix(n, n_cols, rpt, col, val)


@pytest.mark.parametrize("C,sigma", [(32, 64), (32, 512), (32, 1024), (32, 2048), (32, 4096),
                                     (32, 8192), (8, 4096), (64, 2048), (16, 10 ** 9)])
@pytest.mark.parametrize("n", [40_000, 40_000 + 17])
def test_scope_sort_matches_oracle(C, sigma, n):
    m = tie_heavy(n, 6000, seed=n + sigma + C)
    s = sb.crs_to_sell(m, C, sigma)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    for k in ARRAYS:
        assert getattr(s, k).tobytes() == getattr(o, k).tobytes(), (C, sigma, n, k)
    x = np.random.default_rng(1).uniform(-1, 1, m.n_cols)
    assert sb.spmv_sell(s, x).tobytes() == oracle.spmv_sell(o, x).tobytes()


@pytest.mark.parametrize("n,sigma", [(4096, 10 ** 9), (4000, 10 ** 9), (3000, 2048)])
def test_scope_sort_single_window(n, sigma):
    """The whole matrix in one CTA (global scope of <= 4096 rows)."""
    m = tie_heavy(n, 800, seed=3, long_max=40)
    s = sb.crs_to_sell(m, 32, sigma)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, sigma)
    for k in ARRAYS:
        assert getattr(s, k).tobytes() == getattr(o, k).tobytes(), (n, sigma, k)


def test_scope_sort_all_empty_rows():
    n = 5000
    m = CRSMatrix(n, 10, np.zeros(n + 1, np.int64), np.zeros(0, np.int32), np.zeros(0))
    for sigma in (64, 4096, 10 ** 9):
        s = sb.crs_to_sell(m, 32, sigma)
        o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, sigma)
        for k in ARRAYS:
            assert getattr(s, k).tobytes() == getattr(o, k).tobytes(), (sigma, k)


@pytest.mark.parametrize("bad", [-1, 6000, 2 ** 31 - 1])
@pytest.mark.parametrize("permute", [False, True])
def test_device_build_rejects_bad_columns(bad, permute):
    """Device-input builds (crs_to_sell_device: no host-side validation) check
    every column -- inside the fill, or before it when columns are permuted
    -- and raise the reference's StructuralError; the library keeps working."""
    import torch
    m = tie_heavy(6000, 6000, seed=11)
    col = m.col.copy()
    col[len(col) // 2] = bad
    dev = torch.device("cuda", 0)
    rpt_t = torch.from_numpy(m.rpt).to(dev)
    col_t = torch.from_numpy(col).to(dev)
    val_t = torch.from_numpy(m.val).to(dev)
    with pytest.raises(sb.StructuralError, match="column index out of bounds"):
        sb.crs_to_sell_device(rpt_t, col_t, val_t, m.n_rows, m.n_cols, 32, 512,
                              permute_cols=permute)
    good = sb.crs_to_sell_device(rpt_t, torch.from_numpy(m.col).to(dev), val_t, m.n_rows,
                                 m.n_cols, 32, 512, permute_cols=permute)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, 512,
                           permute_cols=permute)
    for k in ARRAYS:
        assert getattr(good, k).tobytes() == getattr(o, k).tobytes(), k


def test_device_build_rejects_decreasing_rpt():
    import torch
    m = tie_heavy(3000, 500, seed=12)
    rpt = m.rpt.copy()
    rpt[100] = rpt[101] + 1
    dev = torch.device("cuda", 0)
    with pytest.raises(sb.StructuralError, match="non-decreasing"):
        sb.crs_to_sell_device(torch.from_numpy(rpt).to(dev), torch.from_numpy(m.col).to(dev),
                              torch.from_numpy(m.val).to(dev), m.n_rows, m.n_cols, 32, 1)
