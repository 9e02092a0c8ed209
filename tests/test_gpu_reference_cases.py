"""The reference's own test intents (pkg/tests/test_formats.py,
test_kernels.py, test_acceptance.py c2/c3/c5), re-expressed against this
package's GPU path.  Each test names the reference test it mirrors.  They
call the public drop-in API (crs_to_sell / spmv_sell / spmv_crs / kernels=),
so a reference user sees the same behaviour on the B200 backend."""

import numpy as np
import pytest

import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import (COOMatrix, DimensionError, ParameterError,
                                  coo_to_crs, crs_to_sell, get_kernels, permute_vector,
                                  spmv_crs, spmv_crs_unrolled, spmv_sell, unpermute_vector)
from conftest import dense_of, random_crs

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


@pytest.fixture
def cuda():
    return get_kernels("cuda")


def four_by_four():
    # rows of lengths 3, 1, 2, 1 (test_formats.py:13-24)
    return coo_to_crs(COOMatrix(4, 4, [0, 0, 0, 1, 2, 2, 3], [0, 1, 2, 1, 0, 3, 2],
                                [1.0, 2, 3, 4, 5, 6, 7]))


class TestLayoutByHand:
    def test_unsorted(self):                       # test_formats.py:90-104
        s = crs_to_sell(four_by_four(), C=2, sigma=1)
        assert (s.n_chunks, s.n_rows_padded, s.stored_slots) == (2, 4, 10)
        assert list(s.cl) == [3, 2] and list(s.cs) == [0, 6, 10]
        assert list(s.perm) == [0, 1, 2, 3]
        assert list(s.val) == [1, 4, 2, 0, 3, 0, 5, 7, 6, 0]
        assert list(s.col) == [0, 1, 1, 0, 2, 0, 0, 2, 3, 0]
        assert sb.chunk_occupancy(s) == pytest.approx(0.7)

    def test_sorted(self):                         # test_formats.py:106-113
        s = crs_to_sell(four_by_four(), C=2, sigma=4)
        assert list(s.perm) == [0, 2, 1, 3]
        assert list(s.cl) == [3, 1] and list(s.cs) == [0, 6, 8]
        assert list(s.val) == [1, 5, 2, 6, 3, 0, 4, 7]
        assert list(s.col) == [0, 0, 1, 3, 2, 0, 1, 2]

    def test_ellpack(self):                        # test_formats.py:115-121
        e = sb.sell_to_ellpack(four_by_four())
        assert e.n_chunks == 1 and e.C == 4 and list(e.cl) == [3]
        assert sb.chunk_occupancy(e) == pytest.approx(7 / 12)

    def test_chunk_one_is_crs(self, rng):          # test_formats.py:130-136
        m = random_crs(rng, 37, 29, 300)
        s = crs_to_sell(m, C=1, sigma=1)
        assert s.val.tobytes() == m.val.tobytes()
        assert s.col.tobytes() == m.col.tobytes()
        assert s.cs.tobytes() == m.rpt.tobytes()

    def test_padding_slots(self, rng):             # test_formats.py:145-153
        s = crs_to_sell(random_crs(rng, 50, 50, 300), C=8, sigma=16)
        cap = np.repeat(s.cl, s.C)
        for p in range(s.n_rows_padded):
            c, r = divmod(p, s.C)
            j = np.arange(s.row_lengths[p], cap[p])
            k = s.cs[c] + j * s.C + r
            assert not s.val[k].any() and not s.col[k].any()


class TestSigma:
    def test_not_multiple_rejected(self, rng):     # test_formats.py:156-159
        with pytest.raises(ParameterError):
            crs_to_sell(random_crs(rng, 100, 100, 500), C=4, sigma=6)

    def test_below_C_is_noop(self, rng):           # test_formats.py:161-168
        m = random_crs(rng, 64, 64, 400)
        a = crs_to_sell(m, 8, 1)
        for sigma in (2, 5, 8):
            b = crs_to_sell(m, 8, sigma)
            assert a.perm.tobytes() == b.perm.tobytes()
            assert a.val.tobytes() == b.val.tobytes()

    def test_at_least_rows_is_global(self, rng):   # test_formats.py:170-177
        m = random_crs(rng, 60, 60, 400)
        perms = [crs_to_sell(m, 8, s).perm.tobytes() for s in (60, 61, 10 ** 6)]
        assert perms[0] == perms[1] == perms[2]

    def test_scope_local(self, rng):               # test_formats.py:179-186
        m = random_crs(rng, 64, 64, 600)
        s = crs_to_sell(m, C=4, sigma=16)
        for k in range(0, 64, 16):
            seg = s.row_lengths[k:k + 16]
            assert (np.diff(seg) <= 0).all()
            assert sorted(seg) == sorted(np.diff(m.rpt)[k:k + 16])

    def test_beta_monotone_in_sigma(self, rng):    # test_acceptance.py:170-189
        m = random_crs(rng, 512, 512, 4000)
        betas = [sb.chunk_occupancy(crs_to_sell(m, 8, s)) for s in (1, 8, 16, 32, 64, 512)]
        assert all(b2 >= b1 for b1, b2 in zip(betas, betas[1:]))

    def test_worst_case_law(self):                 # test_acceptance.py:97-112
        for n_chunks, C in ((1, 2), (8, 4), (64, 16), (8, 32)):
            n = n_chunks * C
            m = coo_to_crs(sb.gen_worst_case(n_chunks, C))
            assert sb.chunk_occupancy(crs_to_sell(m, C, 1)) == (n + C - 1) / (C * n)
            if n_chunks % C == 0:
                assert sb.chunk_occupancy(crs_to_sell(m, C, C * C)) == 1.0


class TestAlignmentAndPermutation:
    def test_alignment(self, rng):                 # test_formats.py:233-241
        m = random_crs(rng, 45, 45, 400)
        s = crs_to_sell(m, C=2, sigma=1, align_bytes=64)
        assert ((s.cs * 4) % 64 == 0).all() and ((s.cl * 4 * s.C) % 64 == 0).all()
        back = sb.sell_to_crs(s)
        assert back.val.tobytes() == m.val.tobytes()

    def test_column_permutation(self, rng, cuda):  # test_kernels.py:132-139
        m = random_crs(rng, 60, 60, 360)
        x = rng.uniform(-1, 1, 60)
        s = crs_to_sell(m, 4, 60, permute_cols=True)
        y = unpermute_vector(spmv_sell(s, permute_vector(x, s.perm), kernels=cuda), s.perm)
        np.testing.assert_allclose(y, dense_of(m) @ x, rtol=1e-12, atol=1e-13)
        back = sb.sell_to_crs(s)
        assert back.col.tobytes() == m.col.tobytes()


class TestKernels:
    @pytest.mark.parametrize("C,sigma", [(1, 1), (2, 2), (4, 16), (8, 64), (16, 16),
                                         (32, 10 ** 9)])
    def test_dense_oracle(self, rng, cuda, C, sigma):   # test_kernels.py:97-106
        m = random_crs(rng, 60, 60, 360)
        x = rng.uniform(-1, 1, 60)
        s = crs_to_sell(m, C, sigma)
        y = unpermute_vector(spmv_sell(s, x, kernels=cuda), s.perm)
        np.testing.assert_allclose(y, dense_of(m) @ x, rtol=1e-12, atol=1e-13)

    def test_crs_and_unrolled(self, rng, cuda):    # test_kernels.py:108-120
        m = random_crs(rng, 60, 60, 360)
        x = rng.uniform(-1, 1, 60)
        ref = dense_of(m) @ x
        np.testing.assert_allclose(spmv_crs(m, x, kernels=cuda), ref, rtol=1e-12, atol=1e-13)
        np.testing.assert_allclose(spmv_crs_unrolled(m, x, kernels=cuda), ref, rtol=1e-12,
                                   atol=1e-13)

    def test_sell_1_1_bitwise_crs(self, rng, cuda):     # test_kernels.py:171-177
        m = random_crs(rng, 81, 81, 486)
        x = rng.uniform(-1, 1, 81)
        assert spmv_sell(crs_to_sell(m, 1, 1), x, kernels=cuda).tobytes() == \
            spmv_crs(m, x, kernels=cuda).tobytes()

    def test_accumulate_once(self, rng, cuda):     # test_kernels.py:181-187
        m = random_crs(rng, 60, 60, 360)
        s = crs_to_sell(m, 8, 32)
        x = rng.uniform(-1, 1, 60)
        y0 = rng.uniform(-1, 1, s.n_rows_padded)
        base = spmv_sell(s, x, kernels=cuda)
        acc = spmv_sell(s, x, y=y0.copy(), accumulate=True, kernels=cuda)
        np.testing.assert_array_equal(acc, y0 + base)

    def test_overwrite_returns_callers_y(self, rng, cuda):   # test_kernels.py:189-195
        s = crs_to_sell(random_crs(rng, 60, 60, 360), 4, 1)
        y = np.full(s.n_rows_padded, 99.0)
        out = spmv_sell(s, np.ones(60), y=y, kernels=cuda)
        assert out is y and not np.any(out == 99.0)

    def test_padded_length_and_zero_rows(self, rng, cuda):   # test_kernels.py:197-209
        s = crs_to_sell(random_crs(rng, 10, 10, 40), 4, 1)
        y = spmv_sell(s, rng.uniform(size=10), kernels=cuda)
        assert y.shape == (12,) and list(y[10:]) == [0.0, 0.0]
        m = coo_to_crs(COOMatrix(4, 4, [0], [2], [3.0]))
        assert list(spmv_sell(crs_to_sell(m, 2, 1), np.ones(4), kernels=cuda)) == \
            [3.0, 0, 0, 0]

    @pytest.mark.parametrize("threads", [2, 3, 8])
    @pytest.mark.parametrize("scheduling", ["static", "guided1"])
    def test_thread_arguments_bitwise(self, rng, cuda, threads, scheduling):
        # test_kernels.py:213-231: results independent of threads/scheduling
        s = crs_to_sell(random_crs(rng, 200, 200, 1200), 8, 32)
        x = rng.uniform(-1, 1, 200)
        ref = spmv_sell(s, x, kernels=cuda)
        y = spmv_sell(s, x, threads=threads, scheduling=scheduling, kernels=cuda)
        assert y.tobytes() == ref.tobytes()

    def test_validation(self, rng, cuda):          # test_kernels.py:271-298
        s = crs_to_sell(random_crs(rng, 5, 5, 15), 4, 1)
        with pytest.raises(DimensionError):
            spmv_sell(s, np.ones(6), kernels=cuda)
        with pytest.raises(DimensionError):
            spmv_sell(s, np.ones(5), y=np.zeros(5), kernels=cuda)
        ro = np.zeros(8)
        ro.flags.writeable = False
        with pytest.raises(ParameterError):
            spmv_sell(s, np.ones(5), y=ro, kernels=cuda)
        assert spmv_sell(s, [1.0, 2, 3, 4, 5], kernels=cuda).tobytes() == \
            spmv_sell(s, np.array([1.0, 2, 3, 4, 5]), kernels=cuda).tobytes()


def test_acceptance_c3_oracle_suite():
    """test_acceptance.py:122-155: 200 random matrices x C x sigma grid vs the
    dense product, tolerance 1e-13 * max(1, N_nzr) * max(1, |ref|_inf)."""
    rng = np.random.default_rng(777)
    for _ in range(200):
        n_rows = int(rng.integers(1, 257))
        n_cols = n_rows if rng.random() < 0.7 else int(rng.integers(1, 257))
        m = random_crs(rng, n_rows, n_cols, int(rng.integers(1, 8 * n_rows + 1)))
        x = rng.uniform(-1, 1, n_cols)
        ref = dense_of(m) @ x
        tol = 1e-13 * max(1.0, m.nnz / n_rows) * max(1.0, float(np.abs(ref).max()))
        assert spmv_sell(crs_to_sell(m, 1, 1), x).tobytes() == spmv_crs(m, x).tobytes()
        for C in (1, 2, 4, 8, 16, 32):
            for sigma in sorted({1, C, 4 * C, n_rows}):
                if C < sigma < n_rows and sigma % C:
                    continue
                s = crs_to_sell(m, C, sigma)
                y = unpermute_vector(spmv_sell(s, x), s.perm)
                assert np.max(np.abs(y - ref)) <= tol
