"""The packed stored-order copy (csrc/sellb_build.cu build_packed, the
row-run kernel k_spmv_rows in MODE 1): pad-heavy C = 32 layouts stream every
row's entries without padding.  The exported SELL arrays are unchanged, and
y is bitwise the oracle's (the reference's _kernels.pyx:65-92 order) with the
copy forced on, off, or chosen by the build's cost model -- overwrite /
accumulate, stored / original order, chunk ranges, fp32, non-finite x[0],
long rows with and without the side table."""

import os
import subprocess
import sys

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, generate

pytestmark = pytest.mark.gpu
ARRAYS = ("cs", "cl", "col", "val", "perm", "row_lengths")


@pytest.fixture(autouse=True)
def _caller_layout(monkeypatch):
    """These tests target the kernels on the caller's own layout: no shadow
    layout (test_gpu_shadow.py covers that one)."""
    monkeypatch.setenv("SELLB_SHADOW", "0")


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


@pytest.mark.parametrize("name", sorted(MATS))
@pytest.mark.parametrize("sigma", [1, 128, 512, 10 ** 9])
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_packed_bitwise(name, sigma, dtype):
    m = MATS[name]()
    if dtype == np.float32:
        m = CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val.astype(np.float32))
    s = sb.crs_to_sell(m, 32, sigma, dtype=dtype)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, sigma)
    x = generate.rhs(m.n_cols).astype(dtype)
    y_ref = oracle.spmv_sell(o, x)
    y0 = np.linspace(-1, 1, s.n_rows_padded).astype(dtype)
    y_acc = y0.copy()
    oracle.spmv_sell_range(o.cs, o.cl, 32, o.col, o.val, x, y_acc, 0, o.n_chunks, True)
    for mode in (True, False, None):
        s.set_packed(mode)
        if mode is True:
            assert s.packed
        for k in ARRAYS:
            assert getattr(s, k).tobytes() == getattr(o, k).tobytes(), (mode, k)
        assert sb.spmv_sell(s, x).tobytes() == y_ref.tobytes(), mode
        assert sb.spmv_sell(s, x, out_order="original").tobytes() == \
            y_ref[o.perm].tobytes(), mode
        assert sb.spmv_sell(s, x, y=y0.copy(), accumulate=True).tobytes() == \
            y_acc.tobytes(), mode


def test_packed_chunk_ranges_and_device_vectors():
    import torch
    from paper_1307_6209_b200 import _lib
    m = MATS["skewed"]()
    s = sb.crs_to_sell(m, 32, 1)
    s.set_packed(True)
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


@pytest.mark.parametrize("x0", [np.inf, -np.inf, np.nan])
def test_packed_nonfinite_x0(x0):
    m = MATS["skewed"]()
    s = sb.crs_to_sell(m, 32, 1)
    s.set_packed(True)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, 1)
    x = generate.rhs(m.n_cols)
    x[0] = x0
    y = sb.spmv_sell(s, x)
    y_ref = oracle.spmv_sell(o, x)
    assert np.array_equal(np.isnan(y), np.isnan(y_ref))
    fin = ~np.isnan(y_ref)
    assert y[fin].tobytes() == y_ref[fin].tobytes()


def test_packed_without_side_table():
    """Long rows read from the SELL arrays (SELLB_LONG_SIDE=0) next to the
    packed short rows (fresh process: the switch is read at build time)."""
    code = (
        "import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
        "import numpy as np, oracle, paper_1307_6209_b200 as sb;"
        "from test_gpu_packed import MATS;"
        "from paper_1307_6209_b200 import generate;"
        "m = MATS['skewed'](); s = sb.crs_to_sell(m, 32, 1); s.set_packed(True);"
        "assert s.long_rows_info()['side_entries'] == 0 and s.long_rows_info()['n_long'] > 0;"
        "o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, 1);"
        "x = generate.rhs(m.n_cols);"
        "assert sb.spmv_sell(s, x).tobytes() == oracle.spmv_sell(o, x).tobytes();"
        "print('ok')")
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, "-c", code], cwd=root, capture_output=True, text=True,
                         env=dict(os.environ, SELLB_LONG_SIDE="0"), timeout=600)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]


def test_packed_cost_model_choices():
    """The cost model (every build's default) packs the pad-heavy unsorted
    layout and leaves dense, sorted and skewed-with-long-rows ones alone."""
    heavy = sb.crs_to_sell(generate.powerlaw(200_000, seed=4, band=5000), 32, 1)
    dense = sb.crs_to_sell(generate.stencil27(32), 32, 1)
    sorted_ = sb.crs_to_sell(generate.powerlaw(200_000, seed=4, band=5000), 32, 10 ** 9)
    skewed = sb.crs_to_sell(sb.coo_to_crs(sb.gen_skewed(1 << 16, 8, 2048, 32)), 32, 1)
    for s in (heavy, dense, sorted_, skewed):
        s.set_packed(None)
    assert heavy.packed and not dense.packed and not sorted_.packed and not skewed.packed
