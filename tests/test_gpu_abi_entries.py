"""Direct C-ABI entry points not exercised through the Python API elsewhere:
the stateless reference-signature range kernel, device CRS kernels, the
membench kernels, and int64 slot offsets beyond 2^31."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import _lib, generate, kernels_cuda
from conftest import case_id, golden_cases, load_case

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


@pytest.mark.parametrize("path", golden_cases()[::4], ids=case_id)
def test_stateless_reference_signature(path):
    """sellb_spmv_sell_range_host: _kernels.pyx:65-68 arguments on host arrays."""
    g = load_case(path)
    lib = _lib.load()
    n = g["n_chunks"]
    for acc, y0, want in ((0, np.zeros(g["n_rows_padded"]), g["y"]),
                          (1, g["y0"].copy(), g["y_acc"])):
        y = y0.copy()
        _lib.check(lib.sellb_spmv_sell_range_host(
            _lib.ptr(g["cs"]), _lib.ptr(g["cl"]), g["C"], _lib.ptr(g["col"]),
            _lib.ptr(g["val"]), len(g["val"]), n, _lib.ptr(g["x"]), len(g["x"]),
            _lib.ptr(y), len(y), 0, n, acc, 0))
        assert y.tobytes() == want.tobytes()


def test_stateless_signature_rejects_bad_range():
    g = load_case(golden_cases()[0])
    lib = _lib.load()
    y = np.zeros(g["n_rows_padded"])
    rc = lib.sellb_spmv_sell_range_host(
        _lib.ptr(g["cs"]), _lib.ptr(g["cl"]), g["C"], _lib.ptr(g["col"]), _lib.ptr(g["val"]),
        len(g["val"]), g["n_chunks"], _lib.ptr(g["x"]), len(g["x"]), _lib.ptr(y), len(y),
        0, g["n_chunks"] + 1, 0, 0)
    assert rc == -1


def test_device_crs_entry():
    """sellb_spmv_crs on device arrays == the reference CRS kernels bitwise."""
    import torch
    m = generate.powerlaw(50_000, seed=6, band=3000)
    x = generate.rhs(m.n_cols)
    t = {k: torch.from_numpy(v).cuda() for k, v in
         (("rpt", m.rpt), ("col", m.col), ("val", m.val), ("x", x))}
    lib = _lib.load()
    for unrolled in (0, 1):
        y = torch.zeros(m.n_rows, dtype=torch.float64, device="cuda")
        _lib.check(lib.sellb_spmv_crs(t["rpt"].data_ptr(), t["col"].data_ptr(),
                                      t["val"].data_ptr(), _lib.SELLB_F64, t["x"].data_ptr(),
                                      y.data_ptr(), 0, m.n_rows, 0, unrolled,
                                      torch.cuda.current_stream().cuda_stream))
        ref = oracle.spmv_crs(m.rpt, m.col, m.val, x, m.n_rows, unrolled=bool(unrolled))
        assert y.cpu().numpy().tobytes() == ref.tobytes()


def test_membench_kernels():
    a = np.random.default_rng(1).uniform(-1, 1, 1_000_003)
    assert kernels_cuda.read_sum(a) == pytest.approx(float(np.sum(a)), rel=1e-12, abs=1e-9)
    dst = np.zeros_like(a)
    kernels_cuda.copy_array(a, dst)
    assert dst.tobytes() == a.tobytes()
    from paper_1307_6209_b200 import membench
    r = membench.microbench_read_sum(n_bytes=256 << 20, reps=3)
    c = membench.microbench_copy(n_bytes=256 << 20, reps=3)
    assert r.gbps > 1000 and c.gbps > 1000


def test_int64_offsets_beyond_2p31_slots():
    """2^27-row cfg5-style matrix: > 2^31 stored slots (int64 cs and flat
    offsets end to end); sampled blocks bit-exact against the oracle."""
    import gc
    import torch
    n = 1 << 27
    free, _ = torch.cuda.mem_get_info()
    if free < 100 << 30:
        pytest.skip("needs ~100 GB of free device memory")
    rpt, col, val = generate.hamiltonian_device(n)
    s = sb.crs_to_sell_device(rpt, col, val, n, n, 32, 1)
    del rpt, col, val
    gc.collect()
    torch.cuda.empty_cache()
    info = s.info()
    assert info.slots > 2 ** 31 and info.nnz > 2 ** 31
    x = generate.rhs(n)
    xd = torch.from_numpy(x).cuda()
    y = sb.spmv_sell(s, xd).cpu().numpy()
    for r0 in (0, n // 2, n - 4096):
        rp, cl_, vl = generate.hamiltonian_rows(n, r0, r0 + 4096)
        o = oracle.crs_to_sell(rp, cl_, vl, 4096, n, 32, 1)
        got = s.export_range(r0 // 32, (r0 + 4096) // 32)
        for k in ("cs", "cl", "col", "val", "row_lengths"):
            assert got[k].tobytes() == getattr(o, k).tobytes(), k
        assert y[r0:r0 + 4096].tobytes() == oracle.spmv_sell(o, x).tobytes()
    s.free()
    del xd
    torch.cuda.empty_cache()


def test_launch_counter_counts_spmv_kernels():
    """sellb_launch_count: one launch per plain SpMV, two for the L2 flush
    (the bench's gpu_launches is built from it)."""
    import torch
    lib = _lib.load()
    m = generate.stencil27(16)
    s = sb.crs_to_sell(m, 32, 1)
    x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
    y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
    sb.spmv_sell(s, x, y)
    a = lib.sellb_launch_count()
    for _ in range(5):
        sb.spmv_sell(s, x, y)
    assert lib.sellb_launch_count() - a == 5
    scratch = torch.empty(1 << 20, dtype=torch.uint8, device="cuda")
    a = lib.sellb_launch_count()
    _lib.check(lib.sellb_l2_flush(scratch.data_ptr(), scratch.numel(),
                                  torch.cuda.current_stream().cuda_stream))
    assert lib.sellb_launch_count() - a == 2


@pytest.mark.parametrize("case", ["n_slots", "col_range", "cl_vs_cs", "cs0", "perm_dup",
                                  "rl_over_cl", "rl_padding"])
def test_import_rejects_inconsistent_layouts(case):
    """sellb_import checks the reference's SellMatrix invariants itself
    (formats.py:210-251) and never reads past the caller's col / val
    (ADVICE r1): every bad layout is SELLB_ESTRUCT, and the library stays
    usable afterwards."""
    import ctypes
    g = next(c for c in map(load_case, golden_cases())
             if c["n_rows_padded"] > c["n_rows"] > 1 and len(c["val"]) and c["cl"][0] > 0)
    lib = _lib.load()
    cs, cl, col, val = g["cs"].copy(), g["cl"].copy(), g["col"].copy(), g["val"].copy()
    perm, rl = g["perm"].copy(), g["row_lengths"].copy()
    n_slots = len(val)
    if case == "n_slots":
        n_slots -= 1
    elif case == "col_range":
        col[len(col) // 2] = g["n_cols"]
    elif case == "cl_vs_cs":
        cl[-1] += 1
    elif case == "cs0":
        cs = cs + g["C"]
    elif case == "perm_dup" and len(perm) > 1:
        perm[1] = perm[0]
    elif case == "rl_over_cl":
        rl[0] = cl[0] + 1
    elif case == "rl_padding":
        rl[-1] = 1 if cl[-1] > 0 else 0
        if rl[-1] == 0:
            pytest.skip("last chunk has width 0")
    out = ctypes.c_void_p()
    rc = lib.sellb_import(_lib.ptr(cs), _lib.ptr(cl), _lib.ptr(col), _lib.ptr(val),
                          _lib.ptr(perm), _lib.ptr(rl), _lib.SELLB_F64, g["n_rows"],
                          g["n_cols"], g["C"], g["sigma"], g["n_chunks"], n_slots, 0, 0,
                          None, 0, ctypes.byref(out))
    assert rc == -3, (case, _lib.last_error())
    assert not out.value
    # the library (and the CUDA context) are still fine
    ok = ctypes.c_void_p()
    _lib.check(lib.sellb_import(_lib.ptr(g["cs"]), _lib.ptr(g["cl"]), _lib.ptr(g["col"]),
                                _lib.ptr(g["val"]), _lib.ptr(g["perm"]),
                                _lib.ptr(g["row_lengths"]), _lib.SELLB_F64, g["n_rows"],
                                g["n_cols"], g["C"], g["sigma"], g["n_chunks"], len(g["val"]),
                                0, 0, None, 0, ctypes.byref(ok)))
    lib.sellb_free(ok.value)
