"""GPU parity: the CUDA path (device build + SpMV kernels, called through the
C ABI) against the reference's golden vectors and the CPU oracle.

Bar: format arrays and permutation bit-exact; fp64 y bit-exact (the kernels
keep the reference's per-row summation order without FMA); fp32 y bit-exact
against the oracle's binary32 loop and within 1e-5 * max(1, |ref|_inf) of
the fp64 reference on the same fp32-representable inputs (BASELINE.json).
"""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, generate, kernels_cuda
from conftest import case_id, golden_cases, load_case, random_crs

pytestmark = pytest.mark.gpu

CASES = golden_cases()
VARIANTS = ("auto", "pad_skip", "pad_incl")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def crs_of(g):
    return CRSMatrix(g["n_rows"], g["n_cols"], g["rpt"], g["col_in"], g["val_in"])


def build(g, **kw):
    return sb.crs_to_sell(crs_of(g), g["C"], g["sigma"], align_bytes=g["align_bytes"],
                          permute_cols=g["permute_cols"], **kw)


def assert_arrays_equal(s, ref):
    get = (lambda k: ref[k]) if isinstance(ref, dict) else (lambda k: getattr(ref, k))
    assert s.n_rows_padded == get("n_rows_padded")
    assert s.n_chunks == get("n_chunks")
    for k in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        a, b = getattr(s, k), get(k)
        assert a.dtype == b.dtype, k
        assert a.tobytes() == b.tobytes(), k


# ---------------------------------------------------------------------------
# golden vectors (produced by the reference itself)
# ---------------------------------------------------------------------------

@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_device_build_bit_exact(path):
    g = load_case(path)
    s = build(g)
    assert_arrays_equal(s, g)
    assert sb.chunk_occupancy(s) == float(g["beta"])


@pytest.mark.parametrize("variant", VARIANTS)
@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_spmv_bitwise(path, variant):
    g = load_case(path)
    s = build(g)
    if variant != "auto":
        s.set_variant(variant)
    y = sb.spmv_sell(s, g["x"])
    assert y.tobytes() == g["y"].tobytes()
    ya = g["y0"].copy()
    out = sb.spmv_sell(s, g["x"], y=ya, accumulate=True)
    assert out is ya
    assert ya.tobytes() == g["y_acc"].tobytes()
    yi = sb.spmv_sell(s, g["x_inf"])           # x[0] = inf: padded rows -> NaN
    np.testing.assert_array_equal(yi, g["y_inf"])


@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_fused_unpermute(path):
    g = load_case(path)
    s = build(g)
    y = sb.spmv_sell(s, g["x"], out_order="original")
    assert y.tobytes() == g["y"][g["perm"]].tobytes()


@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_reference_protocol_range_kernel(path):
    """kernels_cuda.spmv_sell_range with the reference's host arrays and
    argument list (_kernels.pyx:65-68), over split chunk ranges."""
    g = load_case(path)
    n = g["n_chunks"]
    y = np.full(g["n_rows_padded"], 99.0)
    cuts = sorted({0, n // 3, (2 * n) // 3, n})
    for c0, c1 in zip(cuts[:-1], cuts[1:]):
        kernels_cuda.spmv_sell_range(g["cs"], g["cl"], g["C"], g["col"], g["val"],
                                     g["x"], y, c0, c1, False)
    if n:
        assert y.tobytes() == g["y"].tobytes()
    ya = g["y0"].copy()
    kernels_cuda.spmv_sell_range(g["cs"], g["cl"], g["C"], g["col"], g["val"], g["x"],
                                 ya, 0, n, True)
    assert ya.tobytes() == g["y_acc"].tobytes()


@pytest.mark.parametrize("path", CASES[::3], ids=case_id)
def test_host_constructed_sellmatrix(path):
    """A SellMatrix built from host arrays (as the reference dataclass is)
    uploads on first use and multiplies identically."""
    g = load_case(path)
    s = sb.SellMatrix(g["n_rows"], g["n_cols"], g["C"], g["sigma"], g["n_rows_padded"],
                      g["n_chunks"], g["cs"], g["cl"], g["col"], g["val"], g["perm"],
                      g["row_lengths"], g["permute_cols"])
    assert sb.spmv_sell(s, g["x"]).tobytes() == g["y"].tobytes()


@pytest.mark.parametrize("path", CASES, ids=case_id)
def test_crs_kernels_bitwise(path):
    g = load_case(path)
    m = crs_of(g)
    assert sb.spmv_crs(m, g["x"]).tobytes() == g["y_crs"].tobytes()
    assert sb.spmv_crs_unrolled(m, g["x"]).tobytes() == g["y_crs_unrolled"].tobytes()


@pytest.mark.parametrize("path", CASES[::2], ids=case_id)
def test_fp32(path):
    g = load_case(path)
    s = build(g, dtype=np.float32)
    assert s.val.dtype == np.float32
    assert s.val.tobytes() == g["val"].astype(np.float32).tobytes()
    assert s.col.tobytes() == g["col"].tobytes()
    x32 = g["x"].astype(np.float32)
    y = sb.spmv_sell(s, x32)
    ref = oracle.spmv_sell(oracle.OracleSell(
        n_rows_padded=g["n_rows_padded"], n_chunks=g["n_chunks"], C=g["C"],
        cs=g["cs"], cl=g["cl"], col=g["col"], val=g["val"].astype(np.float32)), x32)
    assert y.tobytes() == ref.tobytes()
    # against the fp64 reference on the same fp32-representable inputs
    ref64 = oracle.spmv_sell(oracle.OracleSell(
        n_rows_padded=g["n_rows_padded"], n_chunks=g["n_chunks"], C=g["C"],
        cs=g["cs"], cl=g["cl"], col=g["col"],
        val=g["val"].astype(np.float32).astype(np.float64)), x32.astype(np.float64))
    scale = max(1.0, float(np.abs(ref64).max()) if len(ref64) else 1.0)
    assert np.max(np.abs(y - ref64), initial=0.0) <= 1e-5 * scale


def test_ellpack_and_random_grid(rng):
    """Reference acceptance c3 style: random matrices x C x sigma grid."""
    for i in range(30):
        n_rows = int(rng.integers(1, 257))
        n_cols = n_rows if rng.random() < 0.7 else int(rng.integers(1, 257))
        m = random_crs(rng, n_rows, n_cols, int(rng.integers(1, 8 * n_rows + 1)))
        x = rng.uniform(-1, 1, n_cols)
        for C in (1, 2, 4, 8, 16, 32):
            for sigma in sorted({1, C, 4 * C, max(n_rows, 1)}):
                if C < sigma < n_rows and sigma % C:
                    continue
                s = sb.crs_to_sell(m, C, sigma)
                o = oracle.crs_to_sell(m.rpt, m.col, m.val, n_rows, n_cols, C, sigma)
                assert_arrays_equal(s, vars(o))
                assert sb.spmv_sell(s, x).tobytes() == oracle.spmv_sell(o, x).tobytes()
        e = sb.sell_to_ellpack(m)
        assert e.n_chunks == 1
        back = sb.sell_to_crs(e)
        np.testing.assert_array_equal(back.rpt, m.rpt)
        np.testing.assert_array_equal(back.col, m.col)


# ---------------------------------------------------------------------------
# full BASELINE sizes against the oracle, plus size-independent properties
# ---------------------------------------------------------------------------

def _full_check(m, C, sigma, x, dtype=None):
    s = sb.crs_to_sell(m, C, sigma, dtype=dtype)
    val = m.val if dtype is None else m.val.astype(dtype)
    o = oracle.crs_to_sell(m.rpt, m.col, val, m.n_rows, m.n_cols, C, sigma)
    assert_arrays_equal(s, vars(o))
    xx = x if dtype is None else x.astype(dtype)
    y = sb.spmv_sell(s, xx)
    assert y.tobytes() == oracle.spmv_sell(o, xx, threads=8).tobytes()
    return s, y


@pytest.fixture(scope="module")
def cfg1():
    return generate.laplace2d(1000)


@pytest.fixture(scope="module")
def cfg2():
    return generate.stencil27(128)


def test_cfg1_full(cfg1):
    x = generate.rhs(cfg1.n_cols)
    s, y = _full_check(cfg1, 32, 1, x)
    assert s.nnz == 4_996_000 and s.stored_slots == 4_998_016


def test_cfg2_full_and_properties(cfg2):
    x = generate.rhs(cfg2.n_cols)
    s, y = _full_check(cfg2, 32, 1, x)
    assert s.nnz == 55_742_968 and s.stored_slots == 56_034_816
    # scaling by 2 is exact in binary floating point -> bitwise
    assert sb.spmv_sell(s, 2.0 * x).tobytes() == (2.0 * y).tobytes()
    # determinism across runs and variants
    for v in ("pad_skip", "pad_incl"):
        s.set_variant(v)
        assert sb.spmv_sell(s, x).tobytes() == y.tobytes()
    # linearity within rounding
    x2 = generate.rhs(cfg2.n_cols, seed=7)
    lhs = sb.spmv_sell(s, x + x2)
    rhs = y + sb.spmv_sell(s, x2)
    assert np.max(np.abs(lhs - rhs)) <= 1e-12 * 27 * np.abs(rhs).max()
    # the stencil row sums are known: A @ ones = 26 - (#neighbours)
    ones = sb.spmv_sell(s, np.ones(cfg2.n_cols), out_order="original")
    lens = np.diff(cfg2.rpt)
    np.testing.assert_array_equal(ones, 26.0 - (lens - 1))


def test_cfg2_fp32(cfg2):
    x = generate.rhs(cfg2.n_cols)
    _full_check(cfg2, 32, 1, x, dtype=np.float32)


@pytest.mark.parametrize("sigma", [1, 32, 128, 512, 4_000_000])
def test_cfg3_sigma_sweep(sigma):
    m = _cfg3()
    x = generate.rhs(m.n_cols)
    s, _ = _full_check(m, 32, sigma, x)
    if sigma == 1:
        assert sb.chunk_occupancy(s) < 0.35
    if sigma >= 4_000_000:
        assert sb.chunk_occupancy(s) > 0.95


_CFG3 = {}


def _cfg3():
    if "m" not in _CFG3:
        _CFG3["m"] = generate.powerlaw(4_000_000)
    return _CFG3["m"]


@pytest.mark.parametrize("C", [8, 16, 32, 64, 128])
def test_cfg4_C_sweep(C):
    m = _cfg4()
    x = generate.rhs(m.n_cols)
    for sigma in (1, 4 * C, 16 * C, m.n_rows):
        _full_check(m, C, sigma, x)
    _full_check(m, C, 16 * C, x, dtype=np.float32)


_CFG4 = {}


def _cfg4():
    """BASELINE configs[3] at the size bench.py measures: gen_skewed(2^21,
    base 8, 1024 spikes of 2048) (the reference's generate.py:72-96)."""
    if "m" not in _CFG4:
        _CFG4["m"] = sb.coo_to_crs(sb.gen_skewed(1 << 21, 8, 2048, 1024))
    return _CFG4["m"]


def test_device_input_build_matches_host_input(cfg1):
    import torch
    dev = torch.device("cuda", 0)
    rpt = torch.from_numpy(cfg1.rpt).to(dev)
    col = torch.from_numpy(cfg1.col).to(dev)
    val = torch.from_numpy(cfg1.val).to(dev)
    a = sb.crs_to_sell_device(rpt, col, val, cfg1.n_rows, cfg1.n_cols, 32, 128)
    b = sb.crs_to_sell(cfg1, 32, 128)
    assert_arrays_equal(a, b)


def test_device_tensor_spmv(cfg1):
    import torch
    s = sb.crs_to_sell(cfg1, 32, 1)
    x = generate.rhs(cfg1.n_cols)
    xd = torch.from_numpy(x).cuda()
    yd = sb.spmv_sell(s, xd)
    torch.cuda.synchronize()
    assert yd.cpu().numpy().tobytes() == sb.spmv_sell(s, x).tobytes()


def test_bench_spmv_device_timing(cfg1):
    s = sb.crs_to_sell(cfg1, 32, 1)
    x = generate.rhs(cfg1.n_cols)
    run = sb.bench_spmv(s, x, repetitions=5, trials=3)
    assert run.backend == "cuda" and run.timed_on == "device"
    assert run.flops == 2 * 4_996_000
    assert run.gflops > 1.0
    assert run.checksum == pytest.approx(float(sb.spmv_sell(s, x).sum()), rel=1e-12)


def test_reference_api_with_cuda_kernels():
    """The reference package's own spmv_sell with kernels=cuda (when the
    reference tree is importable, i.e. in the build container)."""
    import os
    import sys
    src = "/root/reference/pkg/src"
    if not os.path.isdir(src):
        pytest.skip("reference tree not present on this host")
    sys.path.insert(0, src)
    try:
        import sellkit
    finally:
        sys.path.remove(src)
    rng = np.random.default_rng(5)
    m = sellkit.coo_to_crs(sellkit.COOMatrix(50, 50, rng.integers(0, 50, 300),
                                             rng.integers(0, 50, 300), rng.uniform(-1, 1, 300)))
    s = sellkit.crs_to_sell(m, 8, 16)
    x = rng.uniform(-1, 1, 50)
    a = sellkit.spmv_sell(s, x, kernels=sb.get_kernels("cuda"))
    b = sellkit.spmv_sell(s, x, kernels=sellkit.get_kernels("python"))
    assert a.tobytes() == b.tobytes()


@pytest.mark.parametrize("n,r0,r1", [(5000, 0, 5000), (1 << 20, 4096, 8192 + 37),
                                     (1 << 22, (1 << 22) - 3000, 1 << 22)])
def test_cfg5_generator_matches_numpy(n, r0, r1):
    """Device generator (csrc/sellb_gen.cu) == NumPy row-addressable definition."""
    rpt_d, col_d, val_d = generate.hamiltonian_device(n, r0, r1)
    rpt, col, val = generate.hamiltonian_rows(n, r0, r1)
    assert rpt_d.cpu().numpy().tobytes() == rpt.tobytes()
    assert col_d.cpu().numpy().tobytes() == col.tobytes()
    assert val_d.cpu().numpy().tobytes() == val.tobytes()


@pytest.mark.parametrize("n,r0,r1,kw", [
    (4_000_000, 0, 4_000_000, {}),                        # the whole cfg3 matrix
    (4_000_000, 1_234_567, 1_300_000, {}),                # a block
    (200_000, 0, 200_000, {"seed": 4, "band": 5000}),
    (5000, 0, 5000, {"lmax": 9000, "mean_base": 40.0}),   # rows capped at n
])
def test_cfg3_generator_matches_numpy(n, r0, r1, kw):
    """Device power-law generator (csrc/sellb_gen.cu k_pl_*) == the NumPy
    row-addressable definition (generate.powerlaw_rows), bit for bit."""
    rpt_d, col_d, val_d = generate.powerlaw_device(n, r0, r1, **kw)
    rpt, col, val = generate.powerlaw_rows(n, r0, r1, **kw)
    assert rpt_d.cpu().numpy().tobytes() == rpt.tobytes()
    assert col_d.cpu().numpy().tobytes() == col.tobytes()
    assert val_d.cpu().numpy().tobytes() == val.tobytes()


def test_cfg5_block_parity_small():
    """Device-generated, device-built matrix: sampled row blocks equal the
    oracle build of the same block regenerated on the host."""
    n = 1 << 20
    rpt_d, col_d, val_d = generate.hamiltonian_device(n)
    s = sb.crs_to_sell_device(rpt_d, col_d, val_d, n, n, 32, 1)
    x = generate.rhs(n)
    y = sb.spmv_sell(s, x)
    for r0 in (0, 1 << 19, n - 4096):
        rpt, col, val = generate.hamiltonian_rows(n, r0, r0 + 4096)
        o = oracle.crs_to_sell(rpt, col, val, 4096, n, 32, 1)
        got = s.export_range(r0 // 32, (r0 + 4096) // 32)
        for k in ("cs", "cl", "col", "val", "row_lengths"):
            assert got[k].tobytes() == getattr(o, k).tobytes(), k
        assert y[r0:r0 + 4096].tobytes() == oracle.spmv_sell(o, x).tobytes()


def test_pipelined_host_path_matches_device(cfg2):
    """sellb_spmv_host's overlapped H2D / compute / D2H path (large matrices)
    equals the device-vector product."""
    import torch
    s = sb.crs_to_sell(cfg2, 32, 1)
    x = generate.rhs(cfg2.n_cols)
    y_host = sb.spmv_sell(s, x)                       # pipelined host path
    y_dev = sb.spmv_sell(s, torch.from_numpy(x).cuda()).cpu().numpy()
    assert y_host.tobytes() == y_dev.tobytes()


def test_tma_path_forced_bitwise():
    """The TMA bulk-copy kernel (sellb_tma.cu) forced on for fp64 too (the
    switch is read once per process, so in a child process): overwrite and
    accumulate results equal the oracle bit for bit."""
    import subprocess
    import sys
    code = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import oracle, paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
m = generate.stencil27(24)
for dt in (np.float64, np.float32):
    s = sb.crs_to_sell(m, 32, 1, dtype=dt)
    s.set_variant("pad_incl")          # the TMA path streams whole chunks
    o = oracle.crs_to_sell(m.rpt, m.col, m.val.astype(dt), m.n_rows, m.n_cols, 32, 1)
    x = generate.rhs(m.n_cols, dtype=dt)
    assert sb.spmv_sell(s, x).tobytes() == oracle.spmv_sell(o, x).tobytes()
    y0 = np.linspace(-1, 1, s.n_rows_padded).astype(dt)
    ya = sb.spmv_sell(s, x, y=y0.copy(), accumulate=True)
    yr = y0.copy()
    oracle.spmv_sell_range(o.cs, o.cl, 32, o.col, o.val, x, yr, 0, o.n_chunks, True)
    assert ya.tobytes() == yr.tobytes()
print("ok")
'''
    import os
    env = dict(os.environ, SELLB_TMA="1")
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         cwd=os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                         timeout=300)
    assert out.returncode == 0 and "ok" in out.stdout, out.stderr[-2000:]
