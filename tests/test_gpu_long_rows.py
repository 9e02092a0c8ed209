"""GPU parity of the long-row paths (sellb_spmv.cu): the row-group kernel
(k_spmv_long_grp, 8-row groups of sorted chunks, producer/chain warps), the
fused warp-per-row role with and without the contiguous side table, and the
packed copy next to them, under every launch mode (SELLB_LONG_MODE 0/1/2)
and wave cap.

Matrices are built so the groups are full, partial (4..7 long rows next to
shorter ones), or sparse (< 4 long rows: warp-per-row), chunks are
homogeneous (threshold 512) or heterogeneous (256), rows are longer than a
batch by ragged amounts, and columns are random (scattered x gathers).  Each
case is checked bit for bit against the CPU oracle: overwrite, accumulate,
fused unpermute, x[0] = inf, fp32, and chunk sub-ranges through the
reference's range-kernel protocol.  The launch knobs are read once per
process, so each mode runs in a child process.
"""

import os
import subprocess
import sys

import numpy as np
import pytest

import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix

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


def long_mix(seed, n=6000, n_cols=50_000):
    """Row lengths: mostly 1..40, plus runs of long rows (600..5000) whose
    counts leave full, partial and sparse 8-row groups after sorting."""
    rng = np.random.default_rng(seed)
    lens = rng.integers(1, 41, n)
    spots = rng.choice(n, 77, replace=False)       # 77 long rows: 9 full groups + 5
    lens[spots] = rng.integers(600, 5001, len(spots))
    lens[rng.choice(n, 9, replace=False)] = rng.integers(257, 520, 9)   # mid-length
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    col = np.concatenate([np.sort(rng.choice(n_cols, L, replace=False)) for L in lens])
    val = rng.uniform(-1, 1, int(rpt[-1]))
    return CRSMatrix(n, n_cols, rpt, col.astype(np.int32), val)


CHILD = r'''
import sys, numpy as np
sys.path.insert(0, ".")
import oracle, paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import kernels_cuda
sys.path.insert(0, "tests")
from test_gpu_long_rows import long_mix
bad = []
for seed in (1, 2):
    m = long_mix(seed)
    for C, sigma in ((32, m.n_rows), (32, 64), (32, 1), (8, m.n_rows), (64, m.n_rows),
                     (128, 256), (4, m.n_rows)):
        for dt in (np.float64, np.float32):
            s = sb.crs_to_sell(m, C, sigma, dtype=dt)
            o = oracle.crs_to_sell(m.rpt, m.col, m.val.astype(dt), m.n_rows, m.n_cols, C, sigma)
            x = np.random.default_rng(seed).uniform(-1, 1, m.n_cols).astype(dt)
            tag = (seed, C, sigma, np.dtype(dt).name)
            if sb.spmv_sell(s, x).tobytes() != oracle.spmv_sell(o, x).tobytes():
                bad.append(("y",) + tag)
            y0 = np.linspace(-1, 1, s.n_rows_padded).astype(dt)
            ya = sb.spmv_sell(s, x, y=y0.copy(), accumulate=True)
            yr = y0.copy()
            oracle.spmv_sell_range(o.cs, o.cl, C, o.col, o.val, x, yr, 0, o.n_chunks, True)
            if ya.tobytes() != yr.tobytes():
                bad.append(("acc",) + tag)
            yo = sb.spmv_sell(s, x, out_order="original")
            ref = oracle.spmv_sell(o, x)[o.perm]
            if yo.tobytes() != ref.tobytes():
                bad.append(("orig",) + tag)
            if dt == np.float64:
                xi = x.copy(); xi[0] = np.inf
                with np.errstate(invalid="ignore"):
                    if sb.spmv_sell(s, xi).tobytes() != oracle.spmv_sell(o, xi).tobytes():
                        bad.append(("inf",) + tag)
                # chunk sub-ranges through the reference's range-kernel protocol
                nc = s.n_chunks
                for c0, c1 in ((0, nc // 3), (nc // 3, nc - 1), (1, 2)):
                    y = np.full(s.n_rows_padded, 7.0)
                    kernels_cuda.spmv_sell_range(s.cs, s.cl, C, s.col, s.val, x, y, c0, c1,
                                                 False)
                    yr = np.full(s.n_rows_padded, 7.0)
                    oracle.spmv_sell_range(o.cs, o.cl, C, o.col, o.val, x, yr, c0, c1, False)
                    if y.tobytes() != yr.tobytes():
                        bad.append(("range", c0, c1) + tag)
            s.free()
print("BAD", bad)
print("ok" if not bad else "fail")
'''

MODES = [
    {"SELLB_LONG_MODE": "2"},                                  # default (side table)
    {"SELLB_LONG_MODE": "2", "SELLB_LONG_GRP": "1"},           # row groups forced
    {"SELLB_LONG_MODE": "0"},
    {"SELLB_LONG_MODE": "1"},
    {"SELLB_LONG_MODE": "1", "SELLB_LONG_GRP": "1"},           # groups, then the bulk
    {"SELLB_LONG_MODE": "2", "SELLB_GRP_CTAS": "3", "SELLB_LONG_GRP": "1"},   # waves of 3
    {"SELLB_LONG_MODE": "2", "SELLB_LONG_SIDE": "0"},           # padded reads, no side table
    {"SELLB_LONG_MODE": "0", "SELLB_LONG_SIDE": "0"},
    {"SELLB_LONG_MODE": "2", "SELLB_PACKED": "1"},              # packed copy + long rows
]


@pytest.mark.parametrize("env", MODES, ids=lambda e: ",".join(f"{k[6:]}={v}" for k, v in e.items()))
def test_long_row_paths_bitwise(env):
    out = subprocess.run([sys.executable, "-c", CHILD], env=dict(os.environ, **env),
                         capture_output=True, text=True, cwd=REPO, timeout=900)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), \
        (out.stdout[-3000:], out.stderr[-3000:])


def test_group_structure_is_exercised():
    """The default build of long_mix really produces full, partial and
    per-row long rows (else the child runs above would test less)."""
    m = long_mix(1)
    rl = sb.crs_to_sell(m, 32, m.n_rows).row_lengths        # sorted: dense groups
    counts = [int((rl[g:g + 8] > 256).sum()) for g in range(0, 96, 8)]
    assert counts.count(8) >= 9 and any(4 <= c < 8 for c in counts)
    rl1 = sb.crs_to_sell(m, 32, 1).row_lengths               # unsorted: isolated rows
    g1 = [int((rl1[g:g + 8] > 256).sum()) for g in range(0, len(rl1), 8)]
    assert any(0 < c < 4 for c in g1)


def test_long_rows_info_reports_the_paths():
    """sellb_long_info: unsorted isolated long rows -> side table, no groups;
    SELLB_LONG_GRP=1 -> row groups (child process: the knob is read at build)."""
    m = long_mix(1)
    info = sb.crs_to_sell(m, 32, 1).long_rows_info()
    assert info["n_long"] > 0 and info["n_groups"] == 0
    assert info["n_rest"] == info["n_long"] and info["side_entries"] > 0
    code = ("import sys; sys.path.insert(0, '.'); sys.path.insert(0, 'tests');"
            "import paper_1307_6209_b200 as sb; from test_gpu_long_rows import long_mix;"
            "m = long_mix(1); print(sb.crs_to_sell(m, 32, m.n_rows).long_rows_info())")
    out = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, SELLB_LONG_GRP="1"),
                         capture_output=True, text=True, cwd=REPO, timeout=300)
    assert out.returncode == 0, out.stderr[-2000:]
    d = eval(out.stdout.strip().splitlines()[-1])
    assert d["n_groups"] >= 9
