"""Seeded fuzz over the build + SpMV parameter space against the CPU oracle:
shapes (n < C, rectangular, empty rows, empty matrix), C in 1..128 (powers of
two and odd heights), sigma in {1, C, k*C, N}, align_bytes {1, 64},
permute_cols (square), fp64 / fp32, both kernel variants, overwrite /
accumulate, stored / original output order, and rows long enough to take the
long-row paths (row groups for C % 8 == 0, warp-per-row otherwise).  Every
case: arrays bit-exact, y bit-exact (binary32 oracle for fp32)."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix

pytestmark = pytest.mark.gpu

ARRAYS = ("cs", "cl", "col", "val", "perm", "row_lengths")


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def random_matrix(rng, n_rows, n_cols, long_rows):
    lens = rng.integers(0, min(n_cols, 24) + 1, n_rows)
    if n_rows and long_rows and n_cols > 300:
        k = rng.choice(n_rows, min(long_rows, n_rows), replace=False)
        lens[k] = rng.integers(257, min(n_cols, 1800) + 1, len(k))
    lens[rng.random(n_rows) < 0.1] = 0                   # empty rows
    rpt = np.zeros(n_rows + 1, np.int64)
    np.cumsum(lens, out=rpt[1:])
    col = (np.concatenate([np.sort(rng.choice(n_cols, L, replace=False)) for L in lens])
           if rpt[-1] else np.zeros(0, np.int64))
    val = rng.uniform(-1, 1, int(rpt[-1]))
    val[rng.random(len(val)) < 0.03] = 0.0               # explicit zeros
    return CRSMatrix(n_rows, n_cols, rpt, col.astype(np.int32), val)


def cases(n):
    rng = np.random.default_rng(20261018)
    out = []
    for i in range(n):
        C = int(rng.choice([1, 2, 3, 4, 5, 7, 8, 12, 16, 24, 32, 48, 64, 96, 128]))
        n_rows = int(rng.choice([0, 1, 5, 31, 33, 257, 1000, 4099, 20000]))
        square = rng.random() < 0.5
        n_cols = n_rows if square else int(rng.choice([1, 17, 500, 3000, 30000]))
        if n_rows == 0:
            n_cols = max(n_cols, 1)
        kinds = [1, C]
        if n_rows > C:
            kinds.append(C * int(rng.integers(2, 9)))
        kinds.append(10 ** 9)
        sigma = int(rng.choice(kinds))
        if C < sigma < n_rows and sigma % C:
            sigma = C
        out.append(dict(seed=i, C=C, n_rows=n_rows, n_cols=max(n_cols, 1), sigma=sigma,
                        align=int(rng.choice([1, 64])),
                        permute=bool(square and n_rows > 0 and rng.random() < 0.4),
                        f32=bool(rng.random() < 0.3),
                        variant=str(rng.choice(["auto", "pad_skip", "pad_incl"])),
                        long_rows=int(rng.choice([0, 0, 3, 40]))))
    return out


CASES = cases(400)


@pytest.mark.parametrize("cs", CASES, ids=lambda c: (
    f"{c['seed']}-C{c['C']}-n{c['n_rows']}x{c['n_cols']}-s{c['sigma']}-a{c['align']}"
    f"{'-p' if c['permute'] else ''}{'-f32' if c['f32'] else ''}-{c['variant']}-L{c['long_rows']}"))
def test_fuzz_build_and_spmv(cs):
    rng = np.random.default_rng(1000 + cs["seed"])
    m = random_matrix(rng, cs["n_rows"], cs["n_cols"], cs["long_rows"])
    dt = np.float32 if cs["f32"] else np.float64
    val = m.val.astype(dt)
    s = sb.crs_to_sell(m, cs["C"], cs["sigma"], align_bytes=cs["align"],
                       permute_cols=cs["permute"], dtype=dt)
    o = oracle.crs_to_sell(m.rpt, m.col, val, m.n_rows, m.n_cols, cs["C"], cs["sigma"],
                           cs["align"], cs["permute"])
    for a in ARRAYS:
        assert getattr(s, a).tobytes() == getattr(o, a).tobytes(), a
    if cs["variant"] != "auto":
        s.set_variant(cs["variant"])
    x = rng.uniform(-1, 1, m.n_cols).astype(dt)
    y = sb.spmv_sell(s, x)
    assert y.tobytes() == oracle.spmv_sell(o, x).tobytes()
    y0 = rng.uniform(-1, 1, s.n_rows_padded).astype(dt)
    ya = sb.spmv_sell(s, x, y=y0.copy(), accumulate=True)
    yr = y0.copy()
    oracle.spmv_sell_range(o.cs, o.cl, cs["C"], o.col, o.val, x, yr, 0, o.n_chunks, True)
    assert ya.tobytes() == yr.tobytes()
    if m.n_rows:
        yo = sb.spmv_sell(s, x, out_order="original")
        assert yo.tobytes() == oracle.spmv_sell(o, x)[o.perm].tobytes()
    s.free()
