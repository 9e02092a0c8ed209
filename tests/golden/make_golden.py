"""Generate the golden parity fixtures from the REFERENCE itself.

Run in the build container (needs /root/reference, which does not exist on
the GPU box):

    make -C oracle ref            # builds oracle/_ref/_kernels*.so
    python tests/golden/make_golden.py

It imports the reference package from /root/reference/pkg/src (its NumPy
`crs_to_sell`, `coo_to_crs`, generators and test fixtures' random-matrix
recipe) and the reference's own compiled kernel core from oracle/_ref, and
writes one small .npz per case into tests/golden/.  The fixtures are
committed; tests/test_oracle_golden.py pins the C oracle to them and the GPU
tests pin the CUDA path to them.
"""

import os
import sys
import importlib.util
import glob
import gzip

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, "/root/reference/pkg/src")
os.environ["SELLKIT_BACKEND"] = "python"

import sellkit  # noqa: E402  (the reference)
from sellkit import (COOMatrix, canonicalize_coo, coo_to_crs, crs_to_sell,  # noqa: E402
                     gen_skewed, gen_worst_case, gen_banded, get_kernels,
                     ParameterError)


def load_ref_compiled():
    hits = glob.glob(os.path.join(REPO, "oracle", "_ref", "_kernels*.so"))
    if not hits:
        raise SystemExit("build oracle/_ref first: make -C oracle ref")
    spec = importlib.util.spec_from_file_location("_kernels", hits[0])
    mod = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mod)
    return mod


def random_coo(rng, n_rows, n_cols, nnz_target, allow_zero_values=False):
    """Reference recipe: pkg/tests/conftest.py:10-23."""
    nnz_target = min(nnz_target, n_rows * n_cols)
    if nnz_target <= 0 or n_rows == 0 or n_cols == 0:
        return COOMatrix(n_rows, n_cols, np.empty(0, np.int32),
                         np.empty(0, np.int32), np.empty(0, np.float64))
    flat = rng.choice(n_rows * n_cols, size=nnz_target, replace=False)
    rows = (flat // n_cols).astype(np.int32)
    cols = (flat % n_cols).astype(np.int32)
    vals = rng.uniform(-1.0, 1.0, size=nnz_target)
    if allow_zero_values:
        vals[rng.random(nnz_target) < 0.05] = 0.0
    return canonicalize_coo(COOMatrix(n_rows, n_cols, rows, cols, vals))


def powerlaw_crs(rng, n, mean_base=4, lmax=150):
    lengths = np.clip(np.floor(mean_base * (1 + rng.pareto(2.0, n))), 1,
                      min(lmax, n)).astype(np.int64)
    rows = np.repeat(np.arange(n), lengths)
    starts = rng.integers(0, n, size=n)
    starts = np.minimum(starts, n - lengths)
    k = np.arange(lengths.sum()) - np.repeat(np.cumsum(lengths) - lengths, lengths)
    cols = np.repeat(starts, lengths) + k
    vals = rng.uniform(-1, 1, len(rows))
    return coo_to_crs(COOMatrix(n, n, rows, cols, vals))


def example_crs():
    """pkg/tests/test_formats.py:13-24."""
    rows = np.array([0, 0, 0, 1, 2, 2, 3], np.int32)
    cols = np.array([0, 1, 2, 1, 0, 3, 2], np.int32)
    vals = np.array([1.0, 2, 3, 4, 5, 6, 7])
    return coo_to_crs(COOMatrix(4, 4, rows, cols, vals))


def cases():
    rng = np.random.default_rng(20240901)
    yield "example_C2_s1", example_crs(), 2, 1, 1, False
    yield "example_C2_s4", example_crs(), 2, 4, 1, False
    m = coo_to_crs(random_coo(rng, 60, 60, 360))
    for C in (1, 2, 4, 8, 16, 32):
        for sigma in sorted({1, C, 4 * C, 60}):
            if C < sigma < 60 and sigma % C:
                continue
            yield f"rand60_C{C}_s{sigma}", m, C, sigma, 1, False
    yield "rand60_C32_sbig", m, 32, 10 ** 9, 1, False
    yield "rect30x70_C8_s16", coo_to_crs(random_coo(rng, 30, 70, 250)), 8, 16, 1, False
    yield "rect70x30_C4_s16", coo_to_crs(random_coo(rng, 70, 30, 400)), 4, 16, 1, False
    mp = coo_to_crs(random_coo(rng, 60, 60, 360))
    yield "permcols_C4_sN", mp, 4, 60, 1, True
    yield "permcols_C8_s16", mp, 8, 16, 1, True
    ma = coo_to_crs(random_coo(rng, 45, 45, 400))
    yield "align64_C2_s1", ma, 2, 1, 64, False
    yield "align64_C4_s8", ma, 4, 8, 64, False
    yield "align64_C3_s1", ma, 3, 1, 64, False
    yield "align64_C32_sN", ma, 32, 45, 64, False
    yield "zeros_C8_s32", coo_to_crs(random_coo(rng, 90, 90, 900, allow_zero_values=True)), 8, 32, 1, False
    rows = np.array([0, 0, 4], np.int32)
    cols = np.array([1, 3, 2], np.int32)
    yield "emptyrows_C2_s5", coo_to_crs(COOMatrix(5, 5, rows, cols, np.array([1.0, 2, 3]))), 2, 5, 1, False
    yield "empty_C2_s1", coo_to_crs(COOMatrix(3, 3, np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0))), 2, 1, 1, False
    yield "zero_rows_C4_s1", coo_to_crs(COOMatrix(0, 5, np.empty(0, np.int32), np.empty(0, np.int32), np.empty(0))), 4, 1, 1, False
    yield "small_n3_C32_s1", coo_to_crs(random_coo(rng, 3, 3, 6)), 32, 1, 1, False
    yield "small_n3_C32_sN", coo_to_crs(random_coo(rng, 3, 3, 6)), 32, 64, 1, False
    yield "ties_C2_s4", coo_to_crs(COOMatrix(4, 1, np.arange(4), np.zeros(4, int), np.ones(4))), 2, 4, 1, False
    wc = coo_to_crs(gen_worst_case(8, 4))
    yield "worst8x4_C4_s1", wc, 4, 1, 1, False
    yield "worst8x4_C4_s16", wc, 4, 16, 1, False
    sk = coo_to_crs(gen_skewed(700, base_len=3, spike_len=200, spike_count=4))
    for sigma in (1, 32, 128, 700):
        yield f"skewed700_C32_s{sigma}", sk, 32, sigma, 1, False
    pl = powerlaw_crs(rng, 1200)
    for C, sigma in ((32, 1), (32, 128), (32, 512), (32, 1200), (8, 64),
                     (16, 256), (64, 256), (128, 512)):
        yield f"powerlaw1200_C{C}_s{sigma}", pl, C, sigma, 1, False
    bd = coo_to_crs(gen_banded(300, 4, fill=0.6))
    yield "banded300_C32_s1", bd, 32, 1, 1, False
    yield "banded300_C32_s64", bd, 32, 64, 1, False


def main():
    comp = load_ref_compiled()
    py = get_kernels("python")
    out_dir = HERE
    for f in glob.glob(os.path.join(out_dir, "case_*.npz")):
        os.remove(f)
    idx = 0
    xrng = np.random.default_rng(12345)
    for name, m, C, sigma, align, permute in cases():
        s = crs_to_sell(m, C, sigma, align_bytes=align, permute_cols=permute)
        x = xrng.uniform(-1, 1, m.n_cols)
        y = np.zeros(s.n_rows_padded)
        comp.spmv_sell_range(s.cs, s.cl, s.C, s.col, s.val, x, y, 0, s.n_chunks, False)
        y_py = np.zeros(s.n_rows_padded)
        py.spmv_sell_range(s.cs, s.cl, s.C, s.col, s.val, x, y_py, 0, s.n_chunks, False)
        assert np.array_equal(y, y_py), name
        y0 = xrng.uniform(-1, 1, s.n_rows_padded)
        y_acc = y0.copy()
        comp.spmv_sell_range(s.cs, s.cl, s.C, s.col, s.val, x, y_acc, 0, s.n_chunks, True)
        # x[0] non-finite: padded slots read x[0] (formats.py:362-363)
        x_inf = x.copy()
        if len(x_inf):
            x_inf[0] = np.inf
        y_inf = np.zeros(s.n_rows_padded)
        with np.errstate(invalid="ignore"):
            comp.spmv_sell_range(s.cs, s.cl, s.C, s.col, s.val, x_inf, y_inf, 0, s.n_chunks, False)
        y_crs = np.zeros(m.n_rows)
        comp.spmv_crs_range(m.rpt, m.col, m.val, x, y_crs, 0, m.n_rows, False)
        y_crs_u = np.zeros(m.n_rows)
        comp.spmv_crs_unrolled_range(m.rpt, m.col, m.val, x, y_crs_u, 0, m.n_rows, False)
        np.savez_compressed(
            os.path.join(out_dir, f"case_{idx:03d}_{name}.npz"),
            name=name, n_rows=m.n_rows, n_cols=m.n_cols, C=C, sigma=sigma,
            align_bytes=align, permute_cols=permute,
            rpt=m.rpt, col_in=m.col, val_in=m.val,
            n_rows_padded=s.n_rows_padded, n_chunks=s.n_chunks,
            cs=s.cs, cl=s.cl, col=s.col, val=s.val, perm=s.perm,
            row_lengths=s.row_lengths, beta=sellkit.chunk_occupancy(s),
            x=x, y=y, y0=y0, y_acc=y_acc, x_inf=x_inf, y_inf=y_inf,
            y_crs=y_crs, y_crs_unrolled=y_crs_u)
        idx += 1
    # parameter-error cases (formats.py:309-332): (n_rows, C, sigma, align)
    m = coo_to_crs(random_coo(np.random.default_rng(5), 100, 100, 500))
    errs = []
    for C, sigma, align, permute in ((4, 6, 1, False), (0, 1, 1, False),
                                     (-2, 1, 1, False), (4, 0, 1, False),
                                     (4, 8, 32, False), (32, 48, 1, False)):
        try:
            crs_to_sell(m, C, sigma, align_bytes=align, permute_cols=permute)
            errs.append((C, sigma, align, 0))
        except ParameterError:
            errs.append((C, sigma, align, 1))
    np.savez_compressed(os.path.join(out_dir, "param_errors.npz"),
                        n_rows=100, cases=np.array(errs, np.int64))
    make_cache_fixtures(out_dir)
    print(f"wrote {idx} cases to {out_dir}")


def make_cache_fixtures(out_dir):
    """.sell files written by the reference's write_sell_cache and the arrays
    its read_sell_cache returns for them (io.py:243-382)."""
    from sellkit import read_sell_cache, write_sell_cache
    rng = np.random.default_rng(31)
    zero_row = COOMatrix(6, 6, [0, 0, 2, 3, 3, 5], [1, 4, 0, 0, 5, 3],
                         [1.5, -2.0, 0.0, 0.0, 7.0, 3.25])   # rows 2/3 end in (0.0, col 0)?
    cases = {
        "rand": (coo_to_crs(random_coo(rng, 60, 60, 360)), 8, 16, False),
        "perm": (coo_to_crs(random_coo(rng, 40, 40, 300)), 4, 40, True),
        "zero_col0": (coo_to_crs(zero_row), 2, 1, False),
    }
    for name, (m, C, sigma, permute) in cases.items():
        s = crs_to_sell(m, C, sigma, permute_cols=permute)
        path = os.path.join(out_dir, f"ref_cache_{name}.sell")
        write_sell_cache(s, path)
        r = read_sell_cache(path)
        np.savez_compressed(os.path.join(out_dir, f"ref_cache_{name}.npz"),
                            n_rows=r.n_rows, n_cols=r.n_cols, C=r.C, sigma=r.sigma,
                            n_rows_padded=r.n_rows_padded, n_chunks=r.n_chunks,
                            col_permuted=r.col_permuted, cs=r.cs, cl=r.cl, col=r.col,
                            val=r.val, perm=r.perm, row_lengths=r.row_lengths,
                            built_row_lengths=s.row_lengths)


def make_coo_fixtures(out_dir):
    """COO -> CRS through the reference's coo_to_crs (formats.py:89-108,
    169-175): unsorted input, duplicate runs of every length class NumPy's
    pairwise summation distinguishes (< 8, 8..128, > 128), signed zeros,
    canonical input (early return), empty rows, empty matrix."""
    rng = np.random.default_rng(77)
    cases = {}
    # many short duplicate runs over a small grid
    n = 4000
    cases["dups_small"] = (50, 40, rng.integers(0, 50, n), rng.integers(0, 40, n),
                           rng.standard_normal(n) * 10.0 ** rng.integers(-6, 6, n))
    # long runs: one coordinate per run length
    lens = [1, 2, 7, 8, 9, 15, 16, 17, 63, 64, 127, 128, 129, 130, 135, 136, 255, 256, 257,
            300, 513, 1000, 2049]
    r = np.concatenate([np.full(L, i % 7) for i, L in enumerate(lens)])
    c = np.concatenate([np.full(L, 3 * i) for i, L in enumerate(lens)])
    v = rng.standard_normal(len(r)) * 10.0 ** rng.integers(-9, 9, len(r))
    p = rng.permutation(len(r))
    cases["dups_long"] = (7, 3 * len(lens), r[p], c[p], v[p])
    # signed zeros and exact cancellation
    cases["zeros"] = (3, 3, [0, 0, 1, 1, 1, 2, 2], [0, 0, 1, 1, 1, 2, 2],
                      [-0.0, -0.0, 0.0, -0.0, -0.0, 1.0, -1.0])
    # canonical already: returned as is
    m = random_coo(rng, 30, 30, 200, allow_zero_values=True)
    cases["canonical"] = (30, 30, m.rows, m.cols, m.vals)
    # unsorted, no duplicates, empty leading/trailing/middle rows
    rows = np.array([9, 3, 3, 5, 9, 3], np.int64)
    cols = np.array([0, 4, 1, 2, 7, 0], np.int64)
    cases["empty_rows"] = (12, 8, rows, cols, rng.standard_normal(6))
    cases["empty"] = (5, 4, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    cases["no_rows"] = (0, 0, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0))
    # a bigger mixed case
    n = 30000
    cases["mixed"] = (3000, 2500, rng.integers(0, 3000, n), rng.integers(0, 2500, n) // 7,
                      rng.uniform(-1, 1, n))
    for name, (nr, nc, rows, cols, vals) in cases.items():
        coo = COOMatrix(nr, nc, np.asarray(rows), np.asarray(cols), np.asarray(vals, float))
        crs = coo_to_crs(coo)
        np.savez_compressed(os.path.join(out_dir, f"coo_{name}.npz"), n_rows=nr, n_cols=nc,
                            rows=coo.rows, cols=coo.cols, vals=coo.vals, rpt=crs.rpt,
                            col=crs.col, val=crs.val)
    # out-of-bounds messages (formats.py:58-70)
    errs = []
    for nr, nc, rows, cols in ((4, 4, [0, 5, -1], [0, 0, 0]), (4, 4, [0, 1], [3, 9]),
                               (4, 4, [2, 7], [9, 0])):
        try:
            COOMatrix(nr, nc, rows, cols, np.ones(len(rows)))
            errs.append("")
        except sellkit.StructuralError as e:
            errs.append(str(e))
    np.savez_compressed(os.path.join(out_dir, "coo_errors.npz"), messages=np.array(errs))


MM_TEXTS = {
    "general": "%%MatrixMarket matrix coordinate real general\n% a comment\n3 4 3\n"
               "1 1 2.5\n2 3 -1e-3\n3 4 7\n",
    "integer": "%%MatrixMarket matrix coordinate integer general\n2 2 2\n1 1 3\n2 2 -4\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n2 2 2\n1 2\n2 1\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n3 3 3\n1 1 5\n2 1 2\n"
                 "3 3 1\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n3 3 2\n2 1 4\n3 2 -1.5\n",
    "skew_diag": "%%MatrixMarket matrix coordinate real skew-symmetric\n2 2 2\n2 1 1\n"
                 "2 2 3\n",
    "duplicates": "%%MatrixMarket matrix coordinate real general\n2 2 4\n1 1 1.5\n2 2 1\n"
                  "1 1 2.25\n1 1 -0.75\n",
    "array_general": "%%MatrixMarket matrix array real general\n2 3\n1\n2\n0\n4\n5\n0\n",
    "array_symmetric": "%%MatrixMarket matrix array real symmetric\n3 3\n1\n2\n3\n4\n"
                       "0\n6\n",
    "array_skew": "%%MatrixMarket matrix array real skew-symmetric\n3 3\n1\n2\n3\n",
    "array_nonsquare_sym": "%%MatrixMarket matrix array real symmetric\n2 3\n1\n2\n3\n",
    "complex": "%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n",
    "hermitian": "%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n",
    "bad_banner": "%%MatrixMarkets matrix coordinate real general\n1 1 1\n1 1 1\n",
    "short_banner": "%%MatrixMarket matrix coordinate real\n1 1 1\n1 1 1\n",
    "bad_object": "%%MatrixMarket vector coordinate real general\n1 1 1\n1 1 1\n",
    "bad_format": "%%MatrixMarket matrix sparse real general\n1 1 1\n1 1 1\n",
    "bad_field": "%%MatrixMarket matrix coordinate double general\n1 1 1\n1 1 1\n",
    "bad_symmetry": "%%MatrixMarket matrix coordinate real diagonal\n1 1 1\n1 1 1\n",
    "pattern_array": "%%MatrixMarket matrix array pattern general\n2 2\n",
    "missing": "%%MatrixMarket matrix coordinate real general\n2 2 3\n1 1 1.0\n",
    "extra": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1.0\n1 1 2.0\n",
    "malformed": "%%MatrixMarket matrix coordinate real general\n% filler comment\n3 3 3\n"
                 "1 1 1.0\n2 oops 2.0\n3 3 3.0\n",
    "token_count": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n"
                   "2 2\n",
    "out_of_range": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n"
                    "3 1 2.0\n",
    "zero_index": "%%MatrixMarket matrix coordinate real general\n2 2 1\n0 1 1.0\n",
    "frac_index": "%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n"
                  "1.5 2 2.0\n",
    "nan_col": "%%MatrixMarket matrix coordinate real general\n2 2 1\n1 nan 1.0\n",
    "bad_size": "%%MatrixMarket matrix coordinate real general\n2 2\n",
    "size_sign": "%%MatrixMarket matrix coordinate real general\n2 -2 1\n",
    "no_size": "%%MatrixMarket matrix coordinate real general\n% only comments\n",
    "empty": "",
    "underscore": "%%MatrixMarket matrix coordinate real general\n1 1 1\n1 1 1_000\n",
    "trailing_comment_then_bad": "%%MatrixMarket matrix coordinate real general\n2 2 2\n"
                                 "1 1 1.0 % note\n2 x 2.0\n",
    "crlf": "%%MatrixMarket matrix coordinate real general\r\n3 3 3\r\n1 1 1.25\r\n"
            "2 2 -2\r\n3 3 1e-300\r\n",
    "tabs_blank_comments": "%%MatrixMarket matrix coordinate real general\n\n%c\n  3\t3  2 \n"
                           "\n1\t2\t+.5e1 % trailing\n% mid\n\n3 1 -7.\n%end\n",
    "specials": "%%MatrixMarket matrix coordinate real general\n2 3 5\n1 1 inf\n1 2 -Infinity\n"
                "2 1 4.9e-324\n2 2 1e400\n2 3 -0.0\n",
    "lone_cr": "%%MatrixMarket matrix coordinate real general\n2 2 2\r1 1 1.0\r2 2 2.0\n",
    "unicode_comment": "%%MatrixMarket matrix coordinate real general\n% caf\u00e9\n1 1 1\n"
                       "1 1 3.5\n",
    "empty_body": "%%MatrixMarket matrix coordinate real general\n4 5 0\n",
}


def make_mm_fixtures(out_dir):
    """read_matrix_market on small texts (results or FormatError messages,
    the path replaced by {path}) and write_matrix_market bytes
    (io.py:192-259)."""
    import tempfile
    from sellkit import FormatError, read_matrix_market, write_matrix_market
    rng = np.random.default_rng(41)
    big = []
    for i in range(4000):
        big.append(f"{rng.integers(1, 301)} {rng.integers(1, 201)} {rng.standard_normal():.17g}")
    texts = dict(MM_TEXTS)
    texts["big"] = "%%MatrixMarket matrix coordinate real general\n300 200 4000\n" + \
        "\n".join(big) + "\n"
    tmp = tempfile.mkdtemp()
    rec = {}
    for name, text in texts.items():
        for gz in (False, True):
            path = os.path.join(tmp, f"{name}.mtx" + (".gz" if gz else ""))
            if gz:
                with gzip.open(path, "wb") as fh:
                    fh.write(text.encode())
            else:
                with open(path, "wb") as fh:
                    fh.write(text.encode())
            key = name + ("_gz" if gz else "")
            try:
                m = read_matrix_market(path)
                rec[key] = dict(ok=True, n_rows=m.n_rows, n_cols=m.n_cols, rows=m.rows,
                                cols=m.cols, vals=m.vals)
            except FormatError as e:
                rec[key] = dict(ok=False, msg=str(e).replace(path, "{path}"))
    np.savez_compressed(os.path.join(out_dir, "mm_read.npz"),
                        names=np.array(sorted(rec)),
                        **{f"text__{k}": np.frombuffer(v.encode(), np.uint8)
                           for k, v in texts.items()},
                        **{f"{k}__{f}": v for k, d in rec.items() for f, v in d.items()})
    # writer bytes
    outs = {}
    cases = {
        "rand": random_coo(rng, 37, 53, 400),
        "dups": COOMatrix(3, 3, [2, 0, 2, 1], [1, 0, 1, 2], [0.1, 1e-300, 0.2, -0.0]),
        "special": COOMatrix(2, 2, [0, 0, 1, 1], [0, 1, 0, 1],
                             [np.inf, -np.inf, np.nan, 5e-324]),
        "empty": COOMatrix(3, 2, np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0)),
    }
    for name, m in cases.items():
        path = os.path.join(tmp, f"w_{name}.mtx")
        write_matrix_market(m, path, comment="written by the reference" if name == "rand"
                            else None)
        outs[f"write__{name}"] = np.frombuffer(open(path, "rb").read(), np.uint8)
        outs[f"coo__{name}__rows"] = m.rows
        outs[f"coo__{name}__cols"] = m.cols
        outs[f"coo__{name}__vals"] = m.vals
        outs[f"coo__{name}__shape"] = np.array(m.shape)
    np.savez_compressed(os.path.join(out_dir, "mm_write.npz"), **outs)


def lru_streams():
    """Line-id streams for the LRU replay (_kernels.pyx:95-139): uniform
    random ids, a cyclic sweep one line larger than some caches (LRU's worst
    case), local reuse with far jumps (many reuse distances just around the
    cache size, exercising the tiled stack-distance path), a single line."""
    rng = np.random.default_rng(95)
    out = {}
    out["uniform"] = (rng.integers(0, 3000, 60000), 3000)
    out["cyclic"] = (np.tile(np.arange(513), 40), 513)
    base = np.repeat(np.arange(0, 20000, 7), 3) % 2600
    jumps = rng.integers(0, 2600, len(base))
    pick = rng.random(len(base)) < 0.3
    out["local_far"] = (np.where(pick, jumps, base), 2600)
    out["single"] = (np.zeros(5000, np.int64), 1)
    out["sparse_ids"] = (rng.integers(0, 40, 9000) * 997, 40 * 997)
    return out


LRU_CACHES = (0, 1, 2, 31, 64, 255, 512, 513, 700, 1500, 2599, 2600, 2999, 3000, 5000)


def make_lru_fixtures(out_dir):
    """Miss counts of the reference's compiled lru_stream_misses and the
    totals of its simulate_rhs_traffic (cachesim.py:49-75) on SELL and CRS
    matrices."""
    comp = load_ref_compiled()
    from sellkit import simulate_rhs_traffic
    arrays = {}
    for name, (lines, slots) in lru_streams().items():
        lines = np.ascontiguousarray(lines, np.int64)
        arrays[f"{name}_lines"] = lines
        arrays[f"{name}_slots"] = np.int64(slots)
        arrays[f"{name}_misses"] = np.array(
            [comp.lru_stream_misses(lines, c, slots) for c in LRU_CACHES], np.int64)
    arrays["caches"] = np.array(LRU_CACHES, np.int64)
    rng = np.random.default_rng(74)
    traffic = []   # (case, C, sigma, cache_bytes, line_bytes, traffic)
    kern = comp
    mats = {0: coo_to_crs(random_coo(rng, 300, 300, 4000)),
            1: coo_to_crs(gen_skewed(700, 4, 120, 9, seed=3)),
            2: coo_to_crs(random_coo(rng, 150, 900, 3000))}
    import sellkit.backend as be
    old = be.kernels
    be.kernels = kern
    try:
        for mi, m in mats.items():
            arrays[f"mat{mi}_rpt"] = m.rpt
            arrays[f"mat{mi}_col"] = m.col
            arrays[f"mat{mi}_val"] = m.val
            arrays[f"mat{mi}_shape"] = np.array([m.n_rows, m.n_cols], np.int64)
            for C, sigma in ((0, 0), (1, 1), (4, 1), (8, 32), (32, 1), (32, 10 ** 9)):
                obj = m if C == 0 else crs_to_sell(m, C, sigma)
                for cache in (0, 64, 512, 4096, 1 << 20):
                    for line in (8, 32, 64, 128):
                        if cache % line:
                            continue
                        v = simulate_rhs_traffic(obj, cache, line, kernels=kern)
                        traffic.append((mi, C, sigma, cache, line, v))
    finally:
        be.kernels = old
    arrays["traffic"] = np.array(traffic, np.int64)
    np.savez_compressed(os.path.join(out_dir, "lru.npz"), **arrays)


if __name__ == "__main__":
    if "--lru-only" in sys.argv:
        make_lru_fixtures(HERE)
    elif "--coo-only" in sys.argv:
        make_coo_fixtures(HERE)
    elif "--mm-only" in sys.argv:
        make_mm_fixtures(HERE)
    else:
        main()
        make_coo_fixtures(HERE)
        make_mm_fixtures(HERE)
        make_lru_fixtures(HERE)
