"""Pin the CPU oracle (oracle/sell_oracle.c) to the reference itself.

The fixtures in tests/golden/ were produced by the reference package
(/root/reference/pkg/src/sellkit, crs_to_sell) and the reference's own
compiled Cython core (oracle/_ref) -- see tests/golden/make_golden.py.  If the
oracle agrees bit for bit here, it is a faithful checker for the GPU tests.
"""

import numpy as np
import pytest

import oracle
from conftest import case_id, golden_cases, load_case

CASES = golden_cases()


def test_fixture_set_is_present():
    assert len(CASES) >= 50


@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_build_bit_exact(path):
    g = load_case(path)
    s = oracle.crs_to_sell(g["rpt"], g["col_in"], g["val_in"], g["n_rows"],
                           g["n_cols"], g["C"], g["sigma"], g["align_bytes"],
                           g["permute_cols"])
    assert s.n_rows_padded == g["n_rows_padded"]
    assert s.n_chunks == g["n_chunks"]
    for k in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        assert getattr(s, k).dtype == g[k].dtype, k
        assert getattr(s, k).tobytes() == g[k].tobytes(), k
    beta = 1.0 if s.stored_slots == 0 else s.nnz / s.stored_slots
    assert beta == float(g["beta"])


@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_spmv_bitwise(path):
    g = load_case(path)
    cs, cl, col, val = g["cs"], g["cl"], g["col"], g["val"]
    y = np.zeros(g["n_rows_padded"])
    oracle.spmv_sell_range(cs, cl, g["C"], col, val, g["x"], y, 0, g["n_chunks"], False)
    assert y.tobytes() == g["y"].tobytes()
    ya = g["y0"].copy()
    oracle.spmv_sell_range(cs, cl, g["C"], col, val, g["x"], ya, 0, g["n_chunks"], True)
    assert ya.tobytes() == g["y_acc"].tobytes()
    yi = np.zeros(g["n_rows_padded"])
    with np.errstate(invalid="ignore"):
        oracle.spmv_sell_range(cs, cl, g["C"], col, val, g["x_inf"], yi, 0,
                               g["n_chunks"], False)
    np.testing.assert_array_equal(yi, g["y_inf"])   # NaN positions included


@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_crs_kernels_bitwise(path):
    g = load_case(path)
    y = oracle.spmv_crs(g["rpt"], g["col_in"], g["val_in"], g["x"], g["n_rows"])
    assert y.tobytes() == g["y_crs"].tobytes()
    yu = oracle.spmv_crs(g["rpt"], g["col_in"], g["val_in"], g["x"], g["n_rows"],
                         unrolled=True)
    assert yu.tobytes() == g["y_crs_unrolled"].tobytes()


def test_threaded_static_split_is_bitwise():
    g = load_case(CASES[-3])
    s = oracle.crs_to_sell(g["rpt"], g["col_in"], g["val_in"], g["n_rows"],
                           g["n_cols"], g["C"], g["sigma"])
    y1 = oracle.spmv_sell(s, g["x"])
    y5 = oracle.spmv_sell(s, g["x"], threads=5)
    assert y1.tobytes() == y5.tobytes()


def test_parameter_errors_match_reference():
    z = np.load(f"{oracle.HERE}/../tests/golden/param_errors.npz")
    n = int(z["n_rows"])
    rpt = np.arange(n + 1, dtype=np.int64)
    col = np.arange(n, dtype=np.int32)
    val = np.ones(n)
    for C, sigma, align, raised in z["cases"]:
        if raised:
            with pytest.raises(ValueError):
                oracle.crs_to_sell(rpt, col, val, n, n, int(C), int(sigma), int(align))
        else:
            oracle.crs_to_sell(rpt, col, val, n, n, int(C), int(sigma), int(align))


def test_read_sum_matches_reference_order():
    a = np.random.default_rng(3).uniform(-1, 1, 1001)
    ref = oracle.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    assert oracle.read_sum(a) == ref.read_sum(a)


@pytest.mark.parametrize("path", CASES[::7], ids=case_id)
def test_reference_core_agrees(path):
    """oracle/_ref (reference source, compiled here) reproduces the goldens."""
    ref = oracle.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    g = load_case(path)
    y = np.zeros(g["n_rows_padded"])
    ref.spmv_sell_range(g["cs"], g["cl"], g["C"], g["col"], g["val"], g["x"], y, 0,
                        g["n_chunks"], False)
    assert y.tobytes() == g["y"].tobytes()
