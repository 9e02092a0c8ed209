"""kernels_cuda.spmv_sell_range (the reference protocol, _kernels.pyx:65-92)
infers row lengths on upload from trailing (0.0, column 0) slots.  Raw SELL
arrays may hold REAL trailing (+-0.0, column 0) entries (the protocol does
not validate column order): their 0*x[0] terms become the single pad term.
Bitwise equal to the reference kernel for finite, infinite and NaN x[0],
overwrite and accumulate, whole and partial chunk ranges."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import kernels_cuda

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def raw_sell(n_chunks, C, n_cols, seed):
    rng = np.random.default_rng(seed)
    cl = rng.integers(0, 12, n_chunks).astype(np.int32)
    cl[rng.random(n_chunks) < 0.05] = rng.integers(200, 600)
    cs = np.zeros(n_chunks + 1, np.int64)
    np.cumsum(C * cl.astype(np.int64), out=cs[1:])
    slots = int(cs[-1])
    col = rng.integers(0, n_cols, slots).astype(np.int32)
    val = rng.uniform(-1, 1, slots)
    for i in range(n_chunks):
        w = int(cl[i])
        for r in range(C):
            ln = int(rng.integers(0, w + 1)) if w else 0
            for j in range(ln, w):                      # the row's padding
                k = cs[i] + j * C + r
                col[k], val[k] = 0, 0.0
            kind = rng.random()
            if ln and kind < 0.15:                      # real trailing (0.0, 0)
                k = cs[i] + (ln - 1) * C + r
                col[k], val[k] = 0, 0.0
            elif ln and kind < 0.25:                    # real trailing (-0.0, 0)
                k = cs[i] + (ln - 1) * C + r
                col[k], val[k] = 0, -0.0
            elif ln > 1 and kind < 0.35:                # (0.0, 0) not at the tail
                k = cs[i] + (ln - 2) * C + r
                col[k], val[k] = 0, 0.0
    return cs, cl, col, val


@pytest.mark.parametrize("C", [32, 8])
@pytest.mark.parametrize("x0", [0.5, -0.25, np.inf, -np.inf, np.nan, -0.0])
def test_protocol_inferred_lengths_bitwise(C, x0):
    n_chunks, n_cols = 3000, 5000
    cs, cl, col, val = raw_sell(n_chunks, C, n_cols, seed=C)
    x = np.random.default_rng(2).uniform(-1, 1, n_cols)
    x[0] = x0
    n = n_chunks * C
    for c0, c1 in ((0, n_chunks), (7, n_chunks - 5), (100, 101)):
        for acc in (False, True):
            y0 = np.linspace(-1, 1, n)
            y_ref = y0.copy()
            oracle.spmv_sell_range(cs, cl, C, col, val, x, y_ref, c0, c1, acc)
            y = y0.copy()
            kernels_cuda.spmv_sell_range(cs, cl, C, col, val, x, y, c0, c1, acc)
            assert y.tobytes() == y_ref.tobytes(), (C, x0, c0, c1, acc)
