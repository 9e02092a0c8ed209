"""COO -> canonical CRS: canonicalize_coo + coo_to_crs
(formats.py:89-108,169-175) and the COOMatrix bounds check (formats.py:50-70).

CPU: the C oracle (oracle_coo_to_crs) and the host mirror are pinned to
fixtures the reference produced (tests/golden/make_golden.py
make_coo_fixtures).  GPU (-m gpu): sellb_coo_to_crs through the host-pointer
entry (coo_to_crs(device=0)), the device-tensor entry (coo_to_crs_device) and
the fused COO -> SELL path, bit-exact against the fixtures and the oracle.
"""

import glob
import os

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200.errors import StructuralError
from conftest import GOLDEN

COO_CASES = sorted(p for p in glob.glob(os.path.join(GOLDEN, "coo_*.npz"))
                   if not p.endswith("coo_errors.npz"))


def cid(p):
    return os.path.basename(p)[4:-4]


def load(p):
    z = np.load(p)
    return {k: z[k] for k in z.files}


def same(a, b):
    return a.dtype == b.dtype and a.tobytes() == b.tobytes()


def test_fixtures_present():
    assert len(COO_CASES) >= 8


@pytest.mark.parametrize("path", COO_CASES, ids=cid)
def test_oracle_pinned_to_reference(path):
    g = load(path)
    rpt, col, val = oracle.coo_to_crs(g["rows"], g["cols"], g["vals"], int(g["n_rows"]))
    assert same(rpt, g["rpt"]) and same(col, g["col"]) and same(val, g["val"])


@pytest.mark.parametrize("path", COO_CASES, ids=cid)
def test_host_mirror_matches_reference(path):
    g = load(path)
    m = sb.coo_to_crs(sb.COOMatrix(int(g["n_rows"]), int(g["n_cols"]), g["rows"], g["cols"],
                                   g["vals"]))
    assert same(m.rpt, g["rpt"]) and same(m.col, g["col"]) and same(m.val, g["val"])


ERR_INPUTS = ((4, 4, [0, 5, -1], [0, 0, 0]), (4, 4, [0, 1], [3, 9]), (4, 4, [2, 7], [9, 0]))


def test_bounds_messages_match_reference():
    want = load(os.path.join(GOLDEN, "coo_errors.npz"))["messages"]
    for (nr, nc, r, c), msg in zip(ERR_INPUTS, want):
        with pytest.raises(StructuralError) as e:
            sb.COOMatrix(nr, nc, r, c, np.ones(len(r)))
        assert str(e.value) == str(msg)


def test_oracle_random_duplicate_heavy_vs_numpy(rng):
    # the restated pairwise sum vs NumPy's own reduceat, at run lengths up to ~1000
    n = 200_000
    rows = rng.integers(0, 40, n)
    cols = rng.integers(0, 5, n)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-12, 12, n)
    rpt, col, val = oracle.coo_to_crs(rows, cols, vals, 40)
    h = sb.coo_to_crs(sb.COOMatrix(40, 5, rows, cols, vals))
    assert same(rpt, h.rpt) and same(col, h.col) and same(val, h.val)


# --------------------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("path", COO_CASES, ids=cid)
def test_gpu_coo_to_crs_matches_reference(path):
    g = load(path)
    m = sb.COOMatrix(int(g["n_rows"]), int(g["n_cols"]), g["rows"], g["cols"], g["vals"])
    h = sb.coo_to_crs(m, device=0)
    assert same(h.rpt, g["rpt"]) and same(h.col, g["col"]) and same(h.val, g["val"])
    d = sb.coo_to_crs_device(m).to_host()
    assert same(d.rpt, g["rpt"]) and same(d.col, g["col"]) and same(d.val, g["val"])


@pytest.mark.gpu
@pytest.mark.parametrize("shape,n", [((1000, 1000), 3_000_000),
                                     ((64, 8), 2_000_000),
                                     ((200_000, 150_000), 4_000_000),
                                     ((3, 2), 100_000)])
def test_gpu_coo_random_vs_oracle(shape, n):
    rng = np.random.default_rng(n + shape[0])
    rows = rng.integers(0, shape[0], n)
    cols = rng.integers(0, shape[1], n)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-10, 10, n)
    rpt, col, val = oracle.coo_to_crs(rows, cols, vals, shape[0])
    h = sb.coo_to_crs(sb.COOMatrix(shape[0], shape[1], rows, cols, vals), device=0)
    assert same(h.rpt, rpt) and same(h.col, col) and same(h.val, val)


@pytest.mark.gpu
def test_gpu_coo_canonical_input_and_stencil_round_trip():
    m = sb.generate.stencil27(32)
    coo = sb.crs_to_coo(m)
    assert coo.is_canonical()
    h = sb.coo_to_crs(coo, device=0)
    assert same(h.rpt, m.rpt) and same(h.col, m.col) and same(h.val, m.val)
    # shuffled copy of the same entries: sorted back to the same CRS
    p = np.random.default_rng(1).permutation(coo.nnz)
    h2 = sb.coo_to_crs(sb.COOMatrix(m.n_rows, m.n_cols, coo.rows[p], coo.cols[p],
                                    coo.vals[p]), device=0)
    assert same(h2.rpt, m.rpt) and same(h2.col, m.col) and same(h2.val, m.val)


@pytest.mark.gpu
def test_gpu_coo_bounds_errors_via_abi():
    import torch
    want = load(os.path.join(GOLDEN, "coo_errors.npz"))["messages"]
    for (nr, nc, r, c), msg in zip(ERR_INPUTS, want):
        t = (nr, nc, torch.tensor(r, dtype=torch.int64, device="cuda"),
             torch.tensor(c, dtype=torch.int64, device="cuda"),
             torch.ones(len(r), dtype=torch.float64, device="cuda"))
        with pytest.raises(StructuralError) as e:
            sb.coo_to_crs_device(t)
        assert str(e.value) == str(msg)


@pytest.mark.gpu
@pytest.mark.parametrize("C,sigma,permute", [(32, 1, False), (8, 64, False), (4, 10**9, True)])
def test_gpu_coo_to_sell_equals_reference_pipeline(C, sigma, permute):
    coo = sb.gen_skewed(20_000, 6, 300, 12, seed=4)
    rng = np.random.default_rng(3)
    extra = 50_000         # add duplicates on top of the generator's entries
    k = rng.integers(0, coo.nnz, extra)
    rows = np.concatenate([coo.rows, coo.rows[k]])
    cols = np.concatenate([coo.cols, coo.cols[k]])
    vals = np.concatenate([coo.vals, rng.uniform(-1, 1, extra)])
    p = rng.permutation(len(rows))
    m = sb.COOMatrix(coo.n_rows, coo.n_cols, rows[p], cols[p], vals[p])
    rpt, col, val = oracle.coo_to_crs(m.rows, m.cols, m.vals, m.n_rows)
    want = oracle.crs_to_sell(rpt, col, val, m.n_rows, m.n_cols, C, sigma, 1, permute)
    s = sb.coo_to_sell(m, C, sigma, permute_cols=permute)
    for a in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        assert same(getattr(s, a), getattr(want, a)), a
