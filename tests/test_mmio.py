"""Matrix Market ingestion / writing against fixtures the
reference produced (tests/golden/make_golden.py make_mm_fixtures, io.py:192-259):
every accepted text gives the reference's triplets bit for bit, every
rejected one the reference's FormatError message and line number, and the
writer the reference's bytes.  The body parser and formatter are host code in
libsellb200.so (no GPU needed); the device canonicalisation and the
file -> SELL path are -m gpu.
"""

import gzip
import os

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import mmio
from paper_1307_6209_b200.errors import FormatError
from conftest import GOLDEN

READ = np.load(os.path.join(GOLDEN, "mm_read.npz"))
WRITE = np.load(os.path.join(GOLDEN, "mm_write.npz"))
NAMES = [str(n) for n in READ["names"]]


def _write(tmp_path, key):
    base = key[:-3] if key.endswith("_gz") else key
    text = READ[f"text__{base}"].tobytes()
    path = str(tmp_path / (base + ".mtx" + (".gz" if key.endswith("_gz") else "")))
    if key.endswith("_gz"):
        with gzip.open(path, "wb") as fh:
            fh.write(text)
    else:
        with open(path, "wb") as fh:
            fh.write(text)
    return path


def same(a, b):
    a, b = np.asarray(a), np.asarray(b)
    return a.dtype == b.dtype and a.shape == b.shape and a.tobytes() == b.tobytes()


def test_fixture_set():
    assert len(NAMES) >= 60


@pytest.mark.parametrize("key", NAMES)
def test_read_matches_reference(tmp_path, key):
    path = _write(tmp_path, key)
    if bool(READ[f"{key}__ok"]):
        m = sb.read_matrix_market(path)
        assert (m.n_rows, m.n_cols) == (int(READ[f"{key}__n_rows"]), int(READ[f"{key}__n_cols"]))
        for f in ("rows", "cols", "vals"):
            assert same(getattr(m, f), READ[f"{key}__{f}"]), f
    else:
        with pytest.raises(FormatError) as e:
            sb.read_matrix_market(path)
        assert str(e.value) == str(READ[f"{key}__msg"]).replace("{path}", path)


@pytest.mark.parametrize("name", ["rand", "dups", "special", "empty"])
def test_write_bytes_match_reference(tmp_path, name):
    shape = WRITE[f"coo__{name}__shape"]
    m = sb.COOMatrix(int(shape[0]), int(shape[1]), WRITE[f"coo__{name}__rows"],
                     WRITE[f"coo__{name}__cols"], WRITE[f"coo__{name}__vals"])
    path = str(tmp_path / "w.mtx")
    sb.write_matrix_market(m, path, comment="written by the reference" if name == "rand"
                           else None)
    assert open(path, "rb").read() == WRITE[f"write__{name}"].tobytes()
    gz = str(tmp_path / "w.mtx.gz")
    sb.write_matrix_market(m, gz, comment="written by the reference" if name == "rand"
                           else None)
    assert gzip.open(gz, "rb").read() == WRITE[f"write__{name}"].tobytes()


def test_round_trip_large_multithreaded(tmp_path, rng):
    """A body large enough to be split across parser threads; round trip is
    exact (%.17g) and equals the NumPy slow path."""
    n = 300_000
    rows = rng.integers(0, 5000, n)
    cols = rng.integers(0, 4000, n)
    vals = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    m = sb.canonicalize_coo(sb.COOMatrix(5000, 4000, rows, cols, vals))
    path = str(tmp_path / "big.mtx")
    sb.write_matrix_market(m, path)
    back = sb.read_matrix_market(path)
    assert same(back.rows, m.rows) and same(back.cols, m.cols) and same(back.vals, m.vals)
    slow = mmio._slow_read(path, 3, 3, m.nnz)
    raw = open(path, "rb").read()
    head = mmio._split_header(raw)
    fast = mmio._parse_body(raw, head[3], 3, m.nnz)
    assert fast is not None and same(fast, slow)


def test_fast_path_declines_what_numpy_would_judge(tmp_path):
    """Exotic tokens go to the NumPy path (so acceptance is NumPy's)."""
    for tok, ok in (("1_000", False), ("0x10", False), ("1d5", False), ("+.5E-3", True),
                    ("-InFiNiTy", True), ("NAN", True)):
        path = str(tmp_path / "t.mtx")
        open(path, "w").write(f"%%MatrixMarket matrix coordinate real general\n1 1 1\n"
                              f"1 1 {tok}\n")
        if ok:
            v = sb.read_matrix_market(path).vals[0]
            ref = float(tok)
            assert (np.isnan(v) and np.isnan(ref)) or v == ref
        else:
            with pytest.raises(FormatError):
                sb.read_matrix_market(path)


# --------------------------------------------------------------------------- GPU

@pytest.mark.gpu
@pytest.mark.parametrize("key", [k for k in NAMES if bool(READ[f"{k}__ok"])])
def test_read_device_canonicalisation(tmp_path, key):
    path = _write(tmp_path, key)
    m = sb.read_matrix_market(path, device=0)
    for f in ("rows", "cols", "vals"):
        assert same(getattr(m, f), READ[f"{key}__{f}"]), f


@pytest.mark.gpu
@pytest.mark.parametrize("C,sigma", [(32, 1), (4, 8), (2, 10**6)])
def test_file_to_sell_on_device(tmp_path, C, sigma):
    path = _write(tmp_path, "big")
    s = sb.read_matrix_market_sell(path, C, sigma)
    rpt, col, val = oracle.coo_to_crs(READ["big__rows"], READ["big__cols"], READ["big__vals"],
                                      int(READ["big__n_rows"]))
    want = oracle.crs_to_sell(rpt, col, val, int(READ["big__n_rows"]),
                              int(READ["big__n_cols"]), C, sigma)
    for a in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        assert same(getattr(s, a), getattr(want, a)), a
