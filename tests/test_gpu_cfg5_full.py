"""Parity at the headline size: BASELINE configs[4], the N = 2^26 banded-
random matrix (1,321,641,891 nonzeros) generated and built on the GPU,
SELL-32-512, fp64 -- the matrix bench.py measures.  The host cannot run the
reference's build on 16 GB of CRS, so the check is block-wise (a block
build equals the slice of the global one when it starts on an
lcm(C, sigma) boundary): the first and the last blocks, and
blocks straddling each quarter boundary (the N = 2 / 4 rank boundaries of
the strong-scaling run), every exported array and y bit-exact against the
oracle (formats.py:295-393, _kernels.pyx:65-92 of the reference; the
reference's own all-grid acceptance check is test_acceptance.py:122-155).
Plus size-independent properties of the whole product."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, generate

pytestmark = pytest.mark.gpu

N = 1 << 26
BLK = 1 << 16
NNZ = 1_321_641_891


@pytest.fixture(scope="module")
def full():
    import torch
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")
    rpt, col, val = generate.hamiltonian_device(N)
    s = sb.crs_to_sell_device(rpt, col, val, N, N, 32, 512)
    del rpt, col, val
    torch.cuda.empty_cache()
    x = np.random.default_rng(12345).uniform(-1, 1, N)
    xd = torch.from_numpy(x).cuda()
    y = sb.spmv_sell(s, xd).cpu().numpy()
    yield s, x, xd, y
    s.free()
    torch.cuda.empty_cache()


def starts():
    out = {0, N - BLK}
    for q in (1, 2, 3):
        b = N * q // 4
        out |= {b - BLK // 2, b}
    return sorted(out)


def test_shape(full):
    s, _, _, _ = full
    assert s.nnz == NNZ and s.n_rows == N and s.n_chunks == N // 32
    assert s.info().variant in (1, 2)


@pytest.mark.parametrize("r0", starts())
def test_block_bit_exact(full, r0):
    s, x, _, y = full
    rp, cl_, vl = generate.hamiltonian_rows(N, r0, r0 + BLK)
    b = CRSMatrix(BLK, N, rp, cl_, vl)
    o = oracle.crs_to_sell(b.rpt, b.col, b.val, BLK, N, 32, 512)
    got = s.export_range(r0 // 32, (r0 + BLK) // 32)
    for k in ("cs", "cl", "col", "val", "row_lengths"):
        assert got[k].tobytes() == getattr(o, k).tobytes(), (r0, k)
    assert y[r0:r0 + BLK].tobytes() == oracle.spmv_sell(o, x).tobytes(), r0


def test_whole_product_properties(full):
    """y(2x) = 2 y(x) bitwise (scaling by 2 is exact), and y(-x) = -y(x)."""
    s, x, xd, y = full
    y2 = sb.spmv_sell(s, 2.0 * xd).cpu().numpy()
    assert y2.tobytes() == (2.0 * y).tobytes()
    yn = sb.spmv_sell(s, -xd).cpu().numpy()
    assert yn.tobytes() == (-y).tobytes()
    assert np.isfinite(y).all()


def test_original_order_epilogue(full):
    """The fused unpermute (out_order="original") equals y[perm] over the
    whole 2^26 rows."""
    s, x, xd, y = full
    yo = sb.spmv_sell(s, xd, out_order="original").cpu().numpy()
    assert yo.tobytes() == y[s.perm].tobytes()
