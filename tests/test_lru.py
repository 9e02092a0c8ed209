"""The LRU replay behind the RHS-traffic simulator (_kernels.pyx:95-139,
cachesim.py:49-75).

CPU: the oracle's restatement against the miss counts the reference's own
compiled core produced (tests/golden/lru.npz, make_golden.py --lru-only) and,
where oracle/_ref is built, against the reference live on fresh streams.
GPU: the device stack-distance count (sellb_lru_stream_misses) against the
oracle on every golden stream x cache size and on larger random streams, and
simulate_rhs_traffic against the reference's totals, plus the reference's
own cachesim laws (tests/test_cachesim.py:44-104 there)."""

import os

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb

HERE = os.path.dirname(os.path.abspath(__file__))
G = np.load(os.path.join(HERE, "golden", "lru.npz"))
STREAMS = ("uniform", "cyclic", "local_far", "single", "sparse_ids")


@pytest.mark.parametrize("name", STREAMS)
def test_oracle_matches_reference_golden(name):
    lines, slots = G[f"{name}_lines"], int(G[f"{name}_slots"])
    got = [oracle.lru_stream_misses(lines, c, slots) for c in G["caches"]]
    assert got == G[f"{name}_misses"].tolist()


def test_oracle_edge_cases():
    assert oracle.lru_stream_misses(np.zeros(0, np.int64), 4, 4) == 0
    assert oracle.lru_stream_misses(np.arange(5), 0, 5) == 5
    assert oracle.lru_stream_misses(np.arange(5), -3, 5) == 5


def test_oracle_vs_reference_live():
    ref = oracle.ref_kernels()
    if ref is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(2024)
    for _ in range(20):
        slots = int(rng.integers(1, 400))
        lines = rng.integers(0, slots, int(rng.integers(0, 5000)))
        for c in (0, 1, slots // 3, slots - 1, slots, slots + 7):
            assert oracle.lru_stream_misses(lines, c, slots) == \
                ref.lru_stream_misses(lines.astype(np.int64), c, slots)


# ---------------------------------------------------------------- GPU ----

gpu = pytest.mark.gpu


@pytest.fixture(scope="module")
def kc():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")
    from paper_1307_6209_b200 import kernels_cuda
    return kernels_cuda


@gpu
@pytest.mark.parametrize("name", STREAMS)
def test_device_matches_golden(kc, name):
    lines, slots = G[f"{name}_lines"], int(G[f"{name}_slots"])
    got = [kc.lru_stream_misses(lines, int(c), slots) for c in G["caches"]]
    assert got == G[f"{name}_misses"].tolist()


@gpu
@pytest.mark.parametrize("seed", range(6))
def test_device_matches_oracle_random(kc, seed):
    """Streams long enough for many whole 1024-position tiles between a
    reuse and its previous access (the tiled binary-search path), with reuse
    distances spread around the cache size."""
    rng = np.random.default_rng(seed)
    slots = int(rng.integers(500, 20000))
    n = int(rng.integers(50000, 400000))
    hot = rng.integers(0, slots, n)
    local = (np.arange(n) // int(rng.integers(1, 9))) % slots
    lines = np.where(rng.random(n) < rng.random(), hot, local).astype(np.int64)
    for c in (1, 7, 100, slots // 8, slots // 2, slots - 1, slots, 2 * slots):
        assert kc.lru_stream_misses(lines, c, slots) == oracle.lru_stream_misses(lines, c, slots)


@gpu
def test_device_edge_cases(kc):
    assert kc.lru_stream_misses(np.zeros(0, np.int64), 4, 4) == 0
    assert kc.lru_stream_misses(np.arange(5), 0, 5) == 5
    assert kc.lru_stream_misses(np.arange(5), -1, 5) == 5
    assert kc.lru_stream_misses(np.zeros(70000, np.int64), 1, 1) == 1
    cyc = np.tile(np.arange(3000), 5)           # LRU worst case: a cycle one too long
    assert kc.lru_stream_misses(cyc, 2999, 3000) == len(cyc)
    assert kc.lru_stream_misses(cyc, 3000, 3000) == 3000
    with pytest.raises(sb.ParameterError):
        kc.lru_stream_misses(np.array([0, 5]), 2, 5)
    with pytest.raises(sb.ParameterError):
        kc.lru_stream_misses(np.array([0, -1]), 2, 5)


def _golden_matrix(mi):
    shape = G[f"mat{mi}_shape"]
    return sb.CRSMatrix(int(shape[0]), int(shape[1]), G[f"mat{mi}_rpt"], G[f"mat{mi}_col"],
                        G[f"mat{mi}_val"])


@gpu
def test_simulate_rhs_traffic_matches_reference(kc):
    built = {}
    for mi, C, sigma, cache, line, want in G["traffic"].tolist():
        key = (mi, C, sigma)
        if key not in built:
            m = _golden_matrix(mi)
            built[key] = m if C == 0 else sb.crs_to_sell(m, C, sigma)
        assert sb.simulate_rhs_traffic(built[key], cache, line, kernels=kc) == want, \
            (mi, C, sigma, cache, line)


@gpu
def test_cachesim_laws(kc):
    """The reference's limiting cases (its test_cachesim.py:44-104)."""
    from paper_1307_6209_b200 import cachesim
    m = sb.coo_to_crs(sb.gen_dense(64))
    # perfect cache: matrix stream + every x line once + y once
    assert cachesim.simulate_rhs_traffic(m, 1 << 20, kernels=kc) == 12 * m.nnz + 8 * 64 + 16 * 64
    # dense rows with a one-line cache: alpha = 1 (one line per 8 entries)
    v = cachesim.simulate_rhs_traffic(m, 64, kernels=kc)
    est = sb.infer_alpha(v, m.nnz, 1.0, m.nnz / m.n_rows, 64)
    assert est.alpha == pytest.approx(1.0, abs=1e-12)
    # traffic non-increasing in the cache size, SELL and CRS alike
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 400, 6000)
    cols = rng.integers(0, 400, 6000)
    c = sb.coo_to_crs(sb.COOMatrix(400, 400, rows, cols, rng.standard_normal(6000)))
    for obj in (c, sb.crs_to_sell(c, 8, 64)):
        t = [cachesim.simulate_rhs_traffic(obj, s, kernels=kc) for s in (0, 64, 640, 6400, 64000)]
        assert all(a >= b for a, b in zip(t, t[1:]))
    # C=1, sigma=1 SELL streams exactly like CRS (no padding)
    s1 = sb.crs_to_sell(c, 1, 1)
    for cache in (0, 512, 4096):
        assert cachesim.simulate_rhs_traffic(s1, cache, kernels=kc) == \
            cachesim.simulate_rhs_traffic(c, cache, kernels=kc)
    with pytest.raises(sb.ParameterError):
        cachesim.simulate_rhs_traffic(m, 1024, line_bytes=48)
    with pytest.raises(sb.ParameterError):
        cachesim.simulate_rhs_traffic(m, 100, line_bytes=64)


@pytest.mark.parametrize("idx", [0, 7, 21, 25, 35, 43, 47, 54])
def test_sell_x_stream_order(idx):
    """The vectorised stream equals the reference's per-chunk walk
    (cachesim.py:31-46) on golden SELL layouts (host arrays only)."""
    from types import SimpleNamespace
    import glob
    from paper_1307_6209_b200.cachesim import sell_x_stream
    path = sorted(glob.glob(os.path.join(HERE, "golden", "case_*.npz")))[idx]
    g = np.load(path)
    m = SimpleNamespace(C=int(g["C"]), n_chunks=int(g["n_chunks"]), cs=g["cs"], cl=g["cl"],
                        col=g["col"], row_lengths=g["row_lengths"])
    want = []
    for i in range(m.n_chunks):
        cl = int(m.cl[i])
        block = m.col[m.cs[i]:m.cs[i] + cl * m.C].reshape(cl, m.C)
        lens = m.row_lengths[i * m.C:(i + 1) * m.C]
        want.extend(block[np.arange(cl)[:, None] < lens[None, :]].tolist())
    assert sell_x_stream(m).tolist() == want


@gpu
@pytest.mark.parametrize("C,sigma", [(1, 1), (4, 1), (8, 64), (32, 1), (64, 10 ** 9), (128, 512)])
def test_device_x_stream_equals_host_stream(kc, C, sigma):
    """sellb_sell_x_lines + device replay == host stream + device replay, on a
    skewed matrix (long rows, empty rows, C > 32 multi-pass lanes)."""
    from types import SimpleNamespace
    from paper_1307_6209_b200 import cachesim
    m = sb.coo_to_crs(sb.gen_skewed(3000, 5, 700, 7, seed=4))
    s = sb.crs_to_sell(m, C, sigma)
    host_only = SimpleNamespace(NAME="host-stream", lru_stream_misses=kc.lru_stream_misses)
    for cache, line in ((0, 64), (512, 32), (4096, 64), (65536, 128), (1 << 22, 64)):
        assert cachesim.simulate_rhs_traffic(s, cache, line, kernels=kc) == \
            cachesim.simulate_rhs_traffic(s, cache, line, kernels=host_only)
