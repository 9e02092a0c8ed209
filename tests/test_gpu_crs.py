"""The CRS kernels of the reference's kernels protocol (_kernels.pyx:17-62)
on the GPU: warp-per-32-rows tiles with coalesced loads and per-row in-order
walks (k_spmv_crs_tiled), bitwise equal to the oracle for the plain and the
unrolled (4 partial sums) kernels -- empty rows, rows spanning many tiles,
ranges not aligned to 32, accumulate, fp32 device arrays -- plus the cached
device handle behind kernels_cuda.spmv_crs_range (uploaded once per buffer)."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, _lib, generate, kernels_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def ragged(seed, n=5000, n_cols=7000):
    rng = np.random.default_rng(seed)
    lens = rng.integers(0, 40, n)
    lens[rng.random(n) < 0.1] = 0
    lens[rng.choice(n, 6, replace=False)] = rng.integers(300, 3000, 6)   # many tiles
    lens = np.minimum(lens, n_cols)
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, L, replace=False)) for L in lens])
    val = rng.uniform(-1, 1, int(rpt[-1]))
    return CRSMatrix(n, n_cols, rpt, col.astype(np.int32), val)


MATS = {"ragged": lambda: ragged(1), "stencil": lambda: generate.stencil27(24),
        "powerlaw": lambda: generate.powerlaw(60_000, seed=2, band=3000),
        "tiny": lambda: ragged(4, n=37, n_cols=50)}


@pytest.mark.parametrize("name", sorted(MATS))
@pytest.mark.parametrize("unrolled", [False, True])
def test_protocol_kernels_bitwise(name, unrolled):
    m = MATS[name]()
    x = generate.rhs(m.n_cols)
    fn = kernels_cuda.spmv_crs_unrolled_range if unrolled else kernels_cuda.spmv_crs_range
    n = m.n_rows
    for r0, r1, acc in ((0, n, False), (0, n, True), (3, n - 5, False), (17, 18, True),
                        (n // 3, 2 * n // 3 + 1, True)):
        if r1 <= r0:
            continue
        y0 = np.linspace(-2, 2, n)
        y = y0.copy()
        fn(m.rpt, m.col, m.val, x, y, r0, r1, acc)
        yr = y0.copy()
        oracle.spmv_crs_range(m.rpt, m.col, m.val, x, yr, r0, r1, acc, unrolled)
        assert y.tobytes() == yr.tobytes(), (name, r0, r1, acc)


def test_handle_is_cached_and_released():
    import gc
    m = ragged(2)
    x = generate.rhs(m.n_cols)
    y = np.zeros(m.n_rows)
    before = len(kernels_cuda._cache)
    for _ in range(3):
        kernels_cuda.spmv_crs_range(m.rpt, m.col, m.val, x, y, 0, m.n_rows, False)
    assert len(kernels_cuda._cache) == before + 1
    del m
    gc.collect()
    assert len(kernels_cuda._cache) == before


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_device_entry_fp32_fp64(dtype):
    import torch
    m = MATS["powerlaw"]()
    x = generate.rhs(m.n_cols).astype(dtype)
    dev = torch.device("cuda", 0)
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).to(dev)
         for k, v in (("rpt", m.rpt), ("col", m.col), ("val", m.val.astype(dtype)), ("x", x))}
    lib = _lib.load()
    code = _lib.SELLB_F32 if dtype == np.float32 else _lib.SELLB_F64
    for unrolled in (0, 1):
        y = torch.zeros(m.n_rows, dtype=t["x"].dtype, device=dev)
        _lib.check(lib.sellb_spmv_crs(t["rpt"].data_ptr(), t["col"].data_ptr(),
                                      t["val"].data_ptr(), code, t["x"].data_ptr(),
                                      y.data_ptr(), 0, m.n_rows, 0, unrolled,
                                      torch.cuda.current_stream().cuda_stream))
        got = y.cpu().numpy()
        if dtype == np.float64:
            ref = oracle.spmv_crs(m.rpt, m.col, m.val, x, m.n_rows, unrolled=bool(unrolled))
            assert got.tobytes() == ref.tobytes()
        else:
            ref = oracle.spmv_crs(m.rpt, m.col, m.val.astype(np.float32).astype(np.float64),
                                  x.astype(np.float64), m.n_rows, unrolled=bool(unrolled))
            assert np.max(np.abs(got - ref)) <= 1e-5 * max(1.0, np.max(np.abs(ref)))


def test_import_rejects_bad_crs():
    import ctypes
    m = ragged(3)
    lib = _lib.load()
    out = ctypes.c_void_p()
    bad = m.col.copy()
    bad[5] = m.n_cols
    rc = lib.sellb_crs_import(_lib.ptr(m.rpt), _lib.ptr(bad), _lib.ptr(m.val), _lib.SELLB_F64,
                              m.n_rows, m.n_cols, len(m.val), 0, ctypes.byref(out))
    assert rc == -3 and not out.value
