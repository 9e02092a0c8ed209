"""The end-to-end host-vector path (spmv_sell with NumPy x / y): pageable
vectors staged through the library's pinned mirrors by its host thread pool,
vectors seen a second time page-locked in place (sellb_host_register) and
released with the array; every variant bit-identical to the device product
and to the oracle (spmv.py:105-122 of the reference is the call)."""

import gc

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, generate, spmv as spmv_mod

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def mat():
    n = 1 << 21                     # x, y = 16.8 MB: above the page-lock threshold
    rp, cl_, vl = generate.hamiltonian_rows(n, 0, n)
    crs = CRSMatrix(n, n, rp, cl_, vl)
    s = sb.crs_to_sell(crs, 32, 512)
    o = oracle.crs_to_sell(crs.rpt, crs.col, crs.val, n, n, 32, 512)
    x = np.random.default_rng(7).uniform(-1, 1, n)
    return s, o, x, oracle.spmv_sell(o, x, threads=8)


def test_pageable_staged_then_registered(mat):
    s, o, x0, y_ref = mat
    x = x0.copy()
    y = np.empty(s.n_rows_padded)
    key = (x.ctypes.data, x.nbytes)
    for call in range(4):
        y[:] = np.nan
        out = sb.spmv_sell(s, x, y)
        assert out is y
        assert y.tobytes() == y_ref.tobytes(), call
        st = spmv_mod._pin_state.get(key)
        assert st == ("seen" if call == 0 else "pinned"), (call, st)
    del x, out
    gc.collect()
    assert key not in spmv_mod._pin_state          # unregistered with the array


def test_y_allocated_per_call_and_small_vectors(mat):
    s, o, x0, y_ref = mat
    for _ in range(3):
        assert sb.spmv_sell(s, x0.copy()).tobytes() == y_ref.tobytes()


def test_views_and_non_owning_buffers(mat):
    s, o, x0, y_ref = mat
    big = np.concatenate([x0, np.zeros(1000)])
    xv = big[: len(x0)]                 # a view: the owner is registered whole
    yb = np.empty(s.n_rows_padded + 7)
    yv = yb[7:]                         # unaligned view into an owned buffer
    for _ in range(3):
        sb.spmv_sell(s, xv, yv)
        assert yv.tobytes() == y_ref.tobytes()
    mv = memoryview(bytearray(x0.tobytes()))   # not NumPy-owned: staged only
    xb = np.frombuffer(mv, dtype=np.float64)
    for _ in range(3):
        assert sb.spmv_sell(s, xb).tobytes() == y_ref.tobytes()


def test_pinned_buffers_through_the_c_abi(mat):
    import ctypes
    from paper_1307_6209_b200 import _lib
    s, o, x0, y_ref = mat
    lib = _lib.load()
    n, m_ = len(x0), s.n_rows_padded
    px, py = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(lib.sellb_host_alloc(n * 8, ctypes.byref(px)))
    _lib.check(lib.sellb_host_alloc(m_ * 8, ctypes.byref(py)))
    try:
        xh = np.ctypeslib.as_array((ctypes.c_double * n).from_address(px.value))
        yh = np.ctypeslib.as_array((ctypes.c_double * m_).from_address(py.value))
        xh[:] = x0
        _lib.check(lib.sellb_spmv_host(s.handle, px.value, py.value, 0, s.n_chunks, 0, 0,
                                       None))
        assert yh.tobytes() == y_ref.tobytes()
    finally:
        lib.sellb_host_free(px)
        lib.sellb_host_free(py)
