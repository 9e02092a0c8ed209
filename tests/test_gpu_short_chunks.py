"""The warp-level variant for very short chunks (k_spmv_sell_short: K chunks
of width <= 2 per warp) and the persistent sweep variant, bit-exact against
the oracle: overwrite, accumulate, original order, pad-skip / pad-inclusive,
ragged tails (n_chunks not a multiple of K), x[0] = inf; knobs are read once
per process, so forced variants run in child processes."""

import os
import subprocess
import sys

import pytest

import paper_1307_6209_b200 as sb

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(autouse=True)
def _caller_layout(monkeypatch):
    """These tests target the kernels on the caller's own layout: no shadow
    layout (test_gpu_shadow.py covers that one)."""
    monkeypatch.setenv("SELLB_SHADOW", "0")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import oracle, paper_1307_6209_b200 as sb
bad = []
rng = np.random.default_rng(7)
for n in (1, 31, 33, 4096 + 32 * 5 + 3, 200_000):
    for wmax in (1, 2, 3):
        lens = rng.integers(0, wmax + 1, n)
        lens[rng.random(n) < 0.5] = wmax
        rpt = np.zeros(n + 1, np.int64); np.cumsum(lens, out=rpt[1:])
        nc = max(n, 8)
        col = np.concatenate([np.sort(rng.choice(nc, L, replace=False)) for L in lens]) \
            if rpt[-1] else np.zeros(0, np.int64)
        m = sb.CRSMatrix(n, nc, rpt, col.astype(np.int32), rng.uniform(-1, 1, int(rpt[-1])))
        for sigma in (1, 64, 10 ** 9):
            for dt in (np.float64, np.float32):
                s = sb.crs_to_sell(m, 32, sigma, dtype=dt)
                o = oracle.crs_to_sell(m.rpt, m.col, m.val.astype(dt), n, nc, 32, sigma)
                for var in ("pad_skip", "pad_incl"):
                    s.set_variant(var)
                    x = rng.uniform(-1, 1, nc).astype(dt)
                    tag = (n, wmax, sigma, np.dtype(dt).name, var)
                    if sb.spmv_sell(s, x).tobytes() != oracle.spmv_sell(o, x).tobytes():
                        bad.append(("y",) + tag)
                    y0 = rng.uniform(-1, 1, s.n_rows_padded).astype(dt)
                    ya = sb.spmv_sell(s, x, y=y0.copy(), accumulate=True)
                    yr = y0.copy()
                    oracle.spmv_sell_range(o.cs, o.cl, 32, o.col, o.val, x, yr, 0, o.n_chunks, True)
                    if ya.tobytes() != yr.tobytes():
                        bad.append(("acc",) + tag)
                    if sb.spmv_sell(s, x, out_order="original").tobytes() != \
                            oracle.spmv_sell(o, x)[o.perm].tobytes():
                        bad.append(("orig",) + tag)
                    if dt == np.float64 and nc:
                        xi = x.copy(); xi[0] = np.inf
                        with np.errstate(invalid="ignore"):
                            if sb.spmv_sell(s, xi).tobytes() != oracle.spmv_sell(o, xi).tobytes():
                                bad.append(("inf",) + tag)
                s.free()
print("BAD", bad[:10])
print("ok" if not bad else "fail")
'''


@pytest.mark.parametrize("env", [{}, {"SELLB_SHORT": "0"}],
                         ids=["default", "off"])
def test_short_chunk_variants_bitwise(env):
    out = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **env),
                         capture_output=True, text=True, cwd=REPO, timeout=900)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), \
        (out.stdout[-3000:], out.stderr[-3000:])
