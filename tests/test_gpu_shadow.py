"""The shadow execution layout (csrc/sellb_build.cu build_shadow, ORD 2 in
csrc/sellb_spmv.cu): irregular layouts run whole-matrix SpMVs on a device
copy of their stored rows re-laid as SELL-32-N (SELL-32-512 when x is far
larger than L2) and scatter each sum back to
the caller's stored / original row.  The exported arrays are unchanged and y
is bitwise the oracle's (the reference's _kernels.pyx:65-92 order for the
CALLER's layout, padding term included) -- every C and sigma, fp32 / fp64,
overwrite / accumulate, both output orders, non-finite x[0], chunk ranges
(which keep the caller's layout)."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, generate

pytestmark = pytest.mark.gpu
ARRAYS = ("cs", "cl", "col", "val", "perm", "row_lengths")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def skewed_rows(rng, n, n_cols, long_frac=0.02):
    lens = np.floor(8.0 / np.sqrt(1.0 - rng.random(n))).astype(np.int64)
    lens = np.minimum(lens, 60)
    k = rng.random(n) < long_frac
    lens[k] = rng.integers(61, 700, int(k.sum()))
    lens[rng.random(n) < 0.05] = 0
    lens = np.minimum(lens, n_cols)
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    starts = rng.integers(0, np.maximum(n_cols - lens, 0) + 1)
    col = (np.repeat(starts, lens) + (np.arange(rpt[-1]) - np.repeat(rpt[:-1], lens)))
    val = rng.uniform(-1, 1, int(rpt[-1]))
    val[rng.random(len(val)) < 0.02] = 0.0
    return CRSMatrix(n, n_cols, rpt, col.astype(np.int32), val)


MATS = {
    "powerlaw": lambda: generate.powerlaw(200_000, seed=4, band=5000),
    "skewed": lambda: skewed_rows(np.random.default_rng(3), 70_001, 90_000),
    "rect": lambda: skewed_rows(np.random.default_rng(5), 5_003, 777, long_frac=0.0),
}


def _check(s, o, x, dtype):
    y_ref = oracle.spmv_sell(o, x)
    y0 = np.linspace(-1, 1, s.n_rows_padded).astype(dtype)
    y_acc = y0.copy()
    oracle.spmv_sell_range(o.cs, o.cl, o.C, o.col, o.val, x, y_acc, 0, o.n_chunks, True)
    assert sb.spmv_sell(s, x).tobytes() == y_ref.tobytes()
    assert sb.spmv_sell(s, x, out_order="original").tobytes() == y_ref[o.perm].tobytes()
    assert sb.spmv_sell(s, x, y=y0.copy(), accumulate=True).tobytes() == y_acc.tobytes()


@pytest.mark.parametrize("name", sorted(MATS))
@pytest.mark.parametrize("C,sigma", [(32, 1), (32, 128), (32, 512), (8, 1), (16, 64),
                                     (64, 1), (128, 2048)])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_shadow_bitwise(name, C, sigma, dtype):
    m = MATS[name]()
    if dtype == np.float32:
        m = CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val.astype(np.float32))
    s = sb.crs_to_sell(m, C, sigma, dtype=dtype)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    x = generate.rhs(m.n_cols).astype(dtype)
    for mode in (True, False, None):
        s.set_shadow(mode)
        if mode is not None:
            assert s.shadow == mode
        for k in ARRAYS:
            assert getattr(s, k).tobytes() == getattr(o, k).tobytes(), (mode, k)
        _check(s, o, x, dtype)


@pytest.mark.parametrize("C,sigma", [(32, 1), (8, 1), (32, 128)])
@pytest.mark.parametrize("x0", [np.inf, -np.inf, np.nan])
def test_shadow_nonfinite_x0(C, sigma, x0):
    """Rows the caller's chunk padded turn NaN (the reference's 0 * x[0]);
    rows the shadow's own chunks pad do not."""
    m = MATS["skewed"]()
    s = sb.crs_to_sell(m, C, sigma)
    s.set_shadow(True)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    x = generate.rhs(m.n_cols)
    x[0] = x0
    for kw, sel in (({}, slice(None)), ({"out_order": "original"}, o.perm)):
        y = sb.spmv_sell(s, x, **kw)
        y_ref = oracle.spmv_sell(o, x)[sel]
        assert np.array_equal(np.isnan(y), np.isnan(y_ref))
        fin = ~np.isnan(y_ref)
        assert y[fin].tobytes() == y_ref[fin].tobytes()


def test_shadow_chunk_ranges_keep_caller_layout():
    import torch
    from paper_1307_6209_b200 import _lib
    m = MATS["skewed"]()
    s = sb.crs_to_sell(m, 32, 1)
    s.set_shadow(True)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, 1)
    x = generate.rhs(m.n_cols)
    xd = torch.from_numpy(x).cuda()
    yd = torch.full((s.n_rows_padded,), 7.0, dtype=torch.float64, device="cuda")
    lib = _lib.load()
    n = s.n_chunks
    cuts = [0, 1, 37, n // 3, n - 5, n]
    for a, b in zip(cuts[:-1], cuts[1:]):
        _lib.check(lib.sellb_spmv(s.handle, xd.data_ptr(), yd.data_ptr(), a, b, 0, 0,
                                  torch.cuda.current_stream().cuda_stream))
    torch.cuda.synchronize()
    assert yd.cpu().numpy().tobytes() == oracle.spmv_sell(o, x).tobytes()


def test_shadow_cost_model_choices(monkeypatch):
    """The byte-level shortlist (SELLB_SHADOW_TIME=0 skips the timed
    decision): irregular layouts get the shadow (SELL-32-N with x in L2);
    dense and already SELL-32-N ones do not."""
    monkeypatch.setenv("SELLB_SHADOW_TIME", "0")
    pl = generate.powerlaw(200_000, seed=4, band=5000)
    heavy = sb.crs_to_sell(pl, 32, 1)
    heavy8 = sb.crs_to_sell(pl, 8, 1)
    dense = sb.crs_to_sell(generate.stencil27(32), 32, 1)
    sorted_ = sb.crs_to_sell(pl, 32, 10 ** 9)
    for s in (heavy, heavy8, dense, sorted_):
        s.set_shadow(None)
    assert heavy.shadow and heavy8.shadow and not dense.shadow and not sorted_.shadow


def test_shadow_from_host_arrays(monkeypatch):
    """A layout uploaded from host arrays (sellb_import, the reference
    dataclass's shape) applies the same cost model and multiplies
    identically."""
    monkeypatch.setenv("SELLB_SHADOW_TIME", "0")
    m = MATS["powerlaw"]()
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, 1)
    s = sb.SellMatrix(o.n_rows, o.n_cols, o.C, o.sigma, o.n_rows_padded, o.n_chunks, o.cs,
                      o.cl, o.col, o.val, o.perm, o.row_lengths, False)
    assert s.shadow
    x = generate.rhs(m.n_cols)
    assert sb.spmv_sell(s, x).tobytes() == oracle.spmv_sell(o, x).tobytes()
    assert sb.spmv_sell(s, x, out_order="original").tobytes() == \
        oracle.spmv_sell(o, x)[o.perm].tobytes()


def test_shadow_empty_rows_and_tiny():
    """All-empty rows, one row, fewer rows than a chunk."""
    for n, n_cols, lens in ((1, 5, [3]), (7, 9, [0, 0, 4, 0, 1, 0, 9]),
                            (40, 40, [0] * 39 + [40]), (33, 12, [0] * 33)):
        rng = np.random.default_rng(n)
        lens = np.asarray(lens, np.int64)
        rpt = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=rpt[1:])
        col = np.concatenate([np.sort(rng.choice(n_cols, k, replace=False))
                              for k in lens] + [np.zeros(0, np.int64)]).astype(np.int32)
        val = rng.uniform(-1, 1, int(rpt[-1]))
        m = CRSMatrix(n, n_cols, rpt, col, val)
        s = sb.crs_to_sell(m, 32, 1)
        o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, 1)
        x = generate.rhs(n_cols)
        if rpt[-1] == 0:
            s.set_shadow(None)
            assert not s.shadow
        else:
            s.set_shadow(True)
            assert s.shadow
        _check(s, o, x, np.float64)


@pytest.mark.parametrize("C,sigma", [(32, 1), (32, 128), (8, 1), (64, 256)])
def test_shadow_windowed_for_large_x(monkeypatch, C, sigma):
    """x larger than SELLB_SHADOW_X_MAX (cfg5's 512 MB x in the library's
    default): the shadow is SELL-32-512, not SELL-32-N, so chunk rows stay
    neighbours; layouts already sorted over >= 512 rows get none.  Bitwise
    either way."""
    monkeypatch.setenv("SELLB_SHADOW_X_MAX", "0")
    monkeypatch.setenv("SELLB_SHADOW_TIME", "0")
    m = MATS["powerlaw"]()
    s = sb.crs_to_sell(m, C, sigma)
    assert s.shadow and s.shadow_sigma == 512
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    _check(s, o, generate.rhs(m.n_cols), np.float64)
    assert not sb.crs_to_sell(m, 32, 512).shadow
    monkeypatch.delenv("SELLB_SHADOW_X_MAX")
    s.set_shadow(None)
    assert s.shadow_sigma >= s.n_rows_padded


@pytest.mark.parametrize("name", sorted(MATS))
@pytest.mark.parametrize("C,sigma", [(32, 1), (8, 1), (32, 512)])
def test_shadow_timed_choice_keeps_results(name, C, sigma):
    """The default cost model settles its shortlist by timing both layouts at
    build time; whichever it keeps, y is the oracle's bit for bit (and a
    re-applied cost model may choose differently without changing y)."""
    m = MATS[name]()
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    x = generate.rhs(m.n_cols)
    s = sb.crs_to_sell(m, C, sigma)
    _check(s, o, x, np.float64)
    s.set_shadow(None)
    _check(s, o, x, np.float64)
