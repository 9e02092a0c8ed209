"""Host-side API: containers, validation order, model closed forms, stats and
generators (CPU only; mirrors the reference's test_formats / test_model /
test_stats cases that need no kernel)."""

import numpy as np
import pytest

import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import (COOMatrix, CRSMatrix, DimensionError,
                                  ParameterError, ResourceError, StructuralError,
                                  generate)
from conftest import random_crs


def example_crs():
    rows = np.array([0, 0, 0, 1, 2, 2, 3])
    cols = np.array([0, 1, 2, 1, 0, 3, 2])
    return sb.coo_to_crs(COOMatrix(4, 4, rows, cols, np.arange(1.0, 8.0)))


class TestContainers:
    def test_canonicalize_sorts_and_sums(self):
        c = sb.canonicalize_coo(COOMatrix(2, 3, [1, 0, 1, 0], [2, 1, 2, 0],
                                          [4.0, 2.0, 6.0, 1.0]))
        assert c.nnz == 3 and c.is_canonical()
        np.testing.assert_array_equal(c.vals, [1.0, 2.0, 10.0])

    def test_coo_bounds(self):
        with pytest.raises(StructuralError):
            COOMatrix(2, 2, [2], [0], [1.0])
        with pytest.raises(StructuralError):
            COOMatrix(2, 2, [0], [0, 1], [1.0])

    def test_crs_validation(self):
        with pytest.raises(StructuralError):
            CRSMatrix(1, 4, [0, 2], [2, 1], [1.0, 2.0])
        with pytest.raises(StructuralError):
            CRSMatrix(2, 4, [0, 3, 2], [0, 1, 2], np.ones(3))
        with pytest.raises(StructuralError):
            CRSMatrix(2, 2, [0, 1, 2], [0, 2], np.ones(2))

    def test_row_restart_allowed(self):
        m = CRSMatrix(2, 3, [0, 2, 4], [0, 2, 0, 1], np.ones(4))
        np.testing.assert_array_equal(m.row_lengths(), [2, 2])

    def test_round_trip(self, rng):
        m = random_crs(rng, 40, 33, 200)
        back = sb.coo_to_crs(sb.crs_to_coo(m))
        np.testing.assert_array_equal(back.rpt, m.rpt)
        np.testing.assert_array_equal(back.col, m.col)
        np.testing.assert_array_equal(back.val, m.val)

    def test_host_sellmatrix_validation(self):
        with pytest.raises(StructuralError):
            sb.SellMatrix(4, 4, 2, 1, 4, 2, [0, 6, 9], [3, 2], np.zeros(10, np.int32),
                          np.zeros(10), [0, 1, 2, 3], [3, 1, 2, 1])
        s = sb.SellMatrix(4, 4, 2, 1, 4, 2, [0, 6, 10], [3, 2], np.zeros(10, np.int32),
                          np.zeros(10), [0, 1, 2, 3], [3, 1, 2, 1])
        assert s.nnz == 7 and s.stored_slots == 10
        assert sb.chunk_occupancy(s) == pytest.approx(0.7)


class TestBuildParameterChecks:
    """Raised before any device work, in the reference's order
    (formats.py:309-332)."""

    def test_C_and_sigma(self, rng):
        m = random_crs(rng, 100, 100, 500)
        for C, sigma in ((0, 1), (-2, 1), (4, 0), (4, 6), (32, 48)):
            with pytest.raises(ParameterError):
                sb.crs_to_sell(m, C, sigma)

    def test_align(self, rng):
        with pytest.raises(ParameterError):
            sb.crs_to_sell(random_crs(rng, 10, 10, 30), 4, 1, align_bytes=32)

    def test_permute_needs_square(self, rng):
        with pytest.raises(ParameterError):
            sb.crs_to_sell(random_crs(rng, 20, 30, 100), 4, 20, permute_cols=True)

    def test_valid_args_need_a_device(self, rng):
        if sb.HAS_CUDA:
            pytest.skip("GPU present")
        with pytest.raises(ResourceError):
            sb.crs_to_sell(random_crs(rng, 10, 10, 30), 4, 1)


class TestVectors:
    def test_permute_round_trip(self):
        perm = np.array([2, 0, 3, 1], np.int32)
        v = np.array([1.0, 2.0, 3.0, 4.0])
        np.testing.assert_array_equal(sb.unpermute_vector(sb.permute_vector(v, perm), perm), v)

    def test_lengths(self):
        with pytest.raises(DimensionError):
            sb.permute_vector(np.ones(3), np.arange(4, dtype=np.int32))
        with pytest.raises(DimensionError):
            sb.unpermute_vector(np.ones(3), np.arange(4, dtype=np.int32))
        assert sb.unpermute_vector(np.ones(6), np.arange(4, dtype=np.int32)).shape == (4,)


class TestBackendSelection:
    def test_cpu_backends_not_shipped(self):
        with pytest.raises(ResourceError):
            sb.get_kernels("compiled")
        with pytest.raises(ParameterError):
            sb.get_kernels("bogus")

    def test_cuda_module_protocol(self):
        from paper_1307_6209_b200 import kernels_cuda as k
        assert k.NAME == "cuda"
        for attr in ("spmv_crs_range", "spmv_crs_unrolled_range", "spmv_sell_range",
                     "lru_stream_misses", "read_sum", "copy_array"):
            assert callable(getattr(k, attr))

    def test_scheduling_validation(self, rng):
        s = sb.SellMatrix(4, 4, 2, 1, 4, 2, [0, 6, 10], [3, 2], np.zeros(10, np.int32),
                          np.zeros(10), [0, 1, 2, 3], [3, 1, 2, 1])
        with pytest.raises(ParameterError):
            sb.spmv_sell(s, np.ones(4), scheduling="dynamic")
        with pytest.raises(ParameterError):
            sb.spmv_sell(s, np.ones(4), threads=0)
        with pytest.raises(DimensionError):
            sb.spmv_sell(s, np.ones(5))
        with pytest.raises(DimensionError):
            sb.spmv_sell(s, np.ones(4), y=np.zeros(3))
        y = np.zeros(4)
        y.flags.writeable = False
        with pytest.raises(ParameterError):
            sb.spmv_sell(s, np.ones(4), y=y)


class TestModel:
    """Closed forms (reference test_model.py / test_acceptance.py:158-167)."""

    def test_balances(self):
        assert sb.code_balance_sell(0.0, 1.0, 1e15) == pytest.approx(6.0, abs=1e-12)
        assert sb.code_balance_crs(0.5, 4) == pytest.approx(6 + 2 + 2)
        assert sb.code_balance_sell(0.5, 0.5, 4) == pytest.approx(12 + 2 + 2)
        assert abs(sb.roofline_upper_bound(43.0, 1.0) - 7.2) <= 0.05
        p = sb.ModelParams(alpha=0.25, beta=1.0, n_nzr=8, n_nzc=8, bandwidth_GBps=100)
        r = sb.roofline(p)
        assert r.predicted_gflops == pytest.approx(100 / (6 + 1 + 1))
        ri = sb.roofline_ideal_alpha(p)
        assert ri.code_balance_bytes_per_flop == pytest.approx(6 + 0.5 + 1)

    def test_infer_alpha_inverts_balance(self):
        nnz, beta, nzr, alpha = 10 ** 6, 0.8, 7.0, 0.3
        v = sb.code_balance_sell(alpha, beta, nzr) * 2 * nnz
        est = sb.infer_alpha(v, nnz, beta, nzr)
        assert est.alpha == pytest.approx(alpha) and est.in_range

    def test_generalised_reduces_to_paper(self):
        assert sb.code_balance_general(0.3, 0.7, 9.0) == pytest.approx(
            sb.code_balance_sell(0.3, 0.7, 9.0))

    def test_algorithmic_bytes_cfg2(self):
        v = sb.algorithmic_bytes(55_742_968, 2_097_152, 2_097_152, 65_536)
        assert v == 703_256_480   # 703.26 MB

    def test_parameter_errors(self):
        with pytest.raises(ParameterError):
            sb.ModelParams(-1, 1, 1, 1, 1)
        with pytest.raises(ParameterError):
            sb.code_balance_sell(0, 0, 1)
        with pytest.raises(ParameterError):
            sb.infer_alpha(1, 1, 1, 1, line_bytes=4)


class TestStatsAndGenerators:
    def test_stats(self):
        m = sb.coo_to_crs(COOMatrix(2, 4, [0, 1, 1, 1], [0, 0, 1, 2], np.ones(4)))
        st = sb.compute_stats(m)
        assert st.zeta == pytest.approx(0.5)
        assert st.footprint_bytes == 12 * 4 + 4 * 3 + 8 * 6

    def test_config_sizes(self):
        m1 = generate.laplace2d(100)
        assert m1.nnz == 5 * 100 * 100 - 4 * 100
        m2 = generate.stencil27(16)
        assert m2.nnz == (3 * 16 - 2) ** 3
        lens = np.diff(m2.rpt)
        assert lens.max() == 27 and lens.min() == 8

    def test_stencil27_128_matches_survey(self):
        # (3*128-2)^3 = 55,742,968
        assert (3 * 128 - 2) ** 3 == 55_742_968

    def test_worst_case_beta_law_inputs(self):
        coo = sb.gen_worst_case(4, 4)
        assert coo.n_rows == 16 and coo.nnz == 4 * 16 + 12

    def test_hamiltonian_is_row_addressable(self):
        n = 5000
        rpt, col, val = generate.hamiltonian_rows(n, 0, n)
        rpt2, col2, val2 = generate.hamiltonian_rows(n, 1000, 2000)
        s, e = rpt[1000], rpt[2000]
        np.testing.assert_array_equal(col[s:e], col2)
        np.testing.assert_array_equal(val[s:e], val2)
        assert (np.abs(val) < 1).all()
        CRSMatrix(n, n, rpt, col, val)   # canonical

    def test_powerlaw_shape(self):
        m = generate.powerlaw(20000)
        lens = np.diff(m.rpt)
        assert 15 < lens.mean() < 25
        st = sb.compute_stats(m)
        assert st.zeta > 0.5
