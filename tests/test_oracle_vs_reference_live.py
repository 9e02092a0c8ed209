"""Live cross-check of the oracle (and the host mirrors) against the reference
package itself, on randomized inputs beyond the committed golden vectors.

Runs only where /root/reference is mounted (the build container; the GPU box
has no reference tree, so it skips there).  It imports the reference's own
Python code -- the checker of the checker -- and compares bit for bit:
crs_to_sell arrays, the SELL product (the reference's Python kernels),
canonicalize_coo / coo_to_crs with duplicates, and the Matrix Market reader
and writer on generated files.
"""

import os
import sys

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference tree not mounted")


@pytest.fixture(scope="module")
def sellkit():
    os.environ.setdefault("SELLKIT_BACKEND", "python")
    sys.path.insert(0, REF)
    try:
        import sellkit as sk
    finally:
        sys.path.remove(REF)
    return sk


def random_coo(rng, sk, n_rows, n_cols, nnz, dups=False):
    rows = rng.integers(0, max(n_rows, 1), nnz) if n_rows else np.zeros(0, np.int64)
    cols = rng.integers(0, max(n_cols, 1), nnz) if n_cols else np.zeros(0, np.int64)
    if not dups and nnz:
        flat = np.unique(rows * max(n_cols, 1) + cols)
        rows, cols = flat // max(n_cols, 1), flat % max(n_cols, 1)
        p = rng.permutation(len(rows))
        rows, cols = rows[p], cols[p]
    vals = rng.standard_normal(len(rows)) * 10.0 ** rng.integers(-6, 6, len(rows))
    vals[rng.random(len(vals)) < 0.05] = 0.0
    return rows, cols, vals


def test_build_and_product_randomized(sellkit):
    rng = np.random.default_rng(99)
    py = sellkit.get_kernels("python")
    for trial in range(150):
        n_rows = int(rng.integers(0, 120))
        square = rng.random() < 0.4
        n_cols = n_rows if square else int(rng.integers(1, 150))
        rows, cols, vals = random_coo(rng, sellkit, n_rows, n_cols,
                                      int(rng.integers(0, 1 + n_rows * 6)))
        ref_m = sellkit.coo_to_crs(sellkit.COOMatrix(n_rows, n_cols, rows, cols, vals))
        C = int(rng.integers(1, 40))
        sig = [1, C, C * int(rng.integers(2, 6)), 10 ** 6][int(rng.integers(0, 4))]
        if C < sig < n_rows and sig % C:
            sig = C
        align = int(rng.choice([1, 64]))
        perm = bool(square and rng.random() < 0.5)
        ref = sellkit.crs_to_sell(ref_m, C, sig, align_bytes=align, permute_cols=perm)
        o = oracle.crs_to_sell(ref_m.rpt, ref_m.col, ref_m.val, n_rows, n_cols, C, sig,
                               align, perm)
        for a in ("cs", "cl", "col", "val", "perm", "row_lengths"):
            assert getattr(o, a).tobytes() == getattr(ref, a).tobytes(), (trial, a)
        x = rng.uniform(-1, 1, n_cols)
        y_ref = np.zeros(ref.n_rows_padded)
        py.spmv_sell_range(ref.cs, ref.cl, ref.C, ref.col, ref.val, x, y_ref, 0,
                           ref.n_chunks, False)
        assert oracle.spmv_sell(o, x).tobytes() == y_ref.tobytes(), trial


def test_coo_canonicalisation_randomized(sellkit):
    rng = np.random.default_rng(5)
    for trial in range(60):
        n_rows, n_cols = int(rng.integers(0, 60)), int(rng.integers(1, 40))
        rows, cols, vals = random_coo(rng, sellkit, n_rows, n_cols,
                                      int(rng.integers(0, 3000)) if n_rows else 0, dups=True)
        ref = sellkit.coo_to_crs(sellkit.COOMatrix(n_rows, n_cols, rows, cols, vals))
        rpt, col, val = oracle.coo_to_crs(rows, cols, vals, n_rows)
        assert rpt.tobytes() == ref.rpt.tobytes(), trial
        assert col.tobytes() == ref.col.astype(np.int32).tobytes(), trial
        assert val.tobytes() == ref.val.tobytes(), trial
        mine = sb.coo_to_crs(sb.COOMatrix(n_rows, n_cols, rows, cols, vals))
        assert mine.val.tobytes() == ref.val.tobytes(), trial


def test_matrix_market_randomized(sellkit, tmp_path):
    rng = np.random.default_rng(11)
    fields = ("real", "integer", "pattern")
    syms = ("general", "symmetric", "skew-symmetric")
    for trial in range(40):
        n = int(rng.integers(1, 30))
        field, sym = fields[trial % 3], syms[(trial // 3) % 3]
        ents = {}
        for _ in range(int(rng.integers(0, n * 3))):
            i, j = int(rng.integers(1, n + 1)), int(rng.integers(1, n + 1))
            if sym != "general" and i < j:
                i, j = j, i
            if sym == "skew-symmetric" and i == j:
                continue
            ents[(i, j)] = rng.standard_normal() * 10.0 ** int(rng.integers(-3, 4))
        lines = [f"%%MatrixMarket matrix coordinate {field} {sym}", "% generated",
                 f"{n} {n} {len(ents)}"]
        for (i, j), v in ents.items():
            if field == "pattern":
                lines.append(f"{i} {j}")
            elif field == "integer":
                lines.append(f"{i} {j} {int(round(v))}")
            else:
                lines.append(f"{i}\t{j}   {v:.{int(rng.integers(3, 18))}g}")
        path = str(tmp_path / f"t{trial}.mtx")
        with open(path, "w") as fh:
            fh.write("\n".join(lines) + "\n")
        a = sellkit.read_matrix_market(path)
        b = sb.read_matrix_market(path)
        assert a.rows.tobytes() == b.rows.tobytes() and a.cols.tobytes() == b.cols.tobytes()
        assert a.vals.tobytes() == b.vals.tobytes(), trial
        p1, p2 = str(tmp_path / "a.mtx"), str(tmp_path / "b.mtx")
        sellkit.write_matrix_market(a, p1, comment="c")
        sb.write_matrix_market(b, p2, comment="c")
        assert open(p1, "rb").read() == open(p2, "rb").read(), trial
