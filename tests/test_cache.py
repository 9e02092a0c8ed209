""".sell cache files (paper_1307_6209_b200/cache.py) against files written by
the reference's own write_sell_cache (tests/golden/ref_cache_*.sell, made by
tests/golden/make_golden.py) -- byte-identical writing, identical reading,
and the reference's FormatError cases (pkg/tests/test_io.py:276-345)."""

import os

import numpy as np
import pytest

import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import FormatError
from paper_1307_6209_b200.cache import read_sell_cache, write_sell_cache
from conftest import GOLDEN

NAMES = ("rand", "perm", "zero_col0")


def ref(name):
    z = np.load(os.path.join(GOLDEN, f"ref_cache_{name}.npz"))
    return {k: z[k] for k in z.files}


def host_matrix(g, row_lengths):
    return sb.SellMatrix(int(g["n_rows"]), int(g["n_cols"]), int(g["C"]), int(g["sigma"]),
                         int(g["n_rows_padded"]), int(g["n_chunks"]), g["cs"], g["cl"],
                         g["col"], g["val"], g["perm"], row_lengths, bool(g["col_permuted"]))


@pytest.mark.parametrize("name", NAMES)
def test_writer_is_byte_identical_to_reference(tmp_path, name):
    g = ref(name)
    out = tmp_path / "m.sell"
    write_sell_cache(host_matrix(g, g["built_row_lengths"]), out)
    assert out.read_bytes() == open(os.path.join(GOLDEN, f"ref_cache_{name}.sell"), "rb").read()


def _corrupt(tmp_path, mutate):
    data = bytearray(open(os.path.join(GOLDEN, "ref_cache_rand.sell"), "rb").read())
    data = mutate(data)
    p = tmp_path / "bad.sell"
    p.write_bytes(bytes(data))
    return p


def test_bad_magic(tmp_path):
    with pytest.raises(FormatError, match="not a chunked-matrix cache"):
        read_sell_cache(_corrupt(tmp_path, lambda d: b"XELL" + d[4:]))


def test_bad_version(tmp_path):
    with pytest.raises(FormatError, match="version 7"):
        read_sell_cache(_corrupt(tmp_path, lambda d: d[:4] + b"\x07\x00" + d[6:]))


def test_truncated(tmp_path):
    for cut in (5, 40, 200, -3):
        with pytest.raises(FormatError, match="truncated"):
            read_sell_cache(_corrupt(tmp_path, lambda d: d[:cut]))


def test_crc(tmp_path):
    def flip(d):
        d[100] ^= 0x40
        return d
    with pytest.raises(FormatError, match="checksum"):
        read_sell_cache(_corrupt(tmp_path, flip))


def test_array_length_check(tmp_path):
    def bad_cl(d):
        # cl count sits after header(56) + cs count(8) + cs data
        import struct
        n_chunks = struct.unpack_from("<Q", d, 48)[0]
        off = 56 + 8 + 8 * (n_chunks + 1)
        struct.pack_into("<Q", d, off, n_chunks + 5)
        return d
    with pytest.raises(FormatError, match="array cl"):
        read_sell_cache(_corrupt(tmp_path, bad_cl))


@pytest.mark.gpu
@pytest.mark.parametrize("name", NAMES)
def test_reader_matches_reference(name):
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")
    g = ref(name)
    s = read_sell_cache(os.path.join(GOLDEN, f"ref_cache_{name}.sell"))
    for k in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        assert getattr(s, k).tobytes() == g[k].tobytes(), k
    assert s.col_permuted == bool(g["col_permuted"])
    assert s.nnz == int(g["row_lengths"].sum())


@pytest.mark.gpu
def test_device_round_trip(tmp_path):
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")
    from paper_1307_6209_b200 import generate
    m = generate.powerlaw(50_000, seed=8, band=2000)
    s = sb.crs_to_sell(m, 32, 256)
    write_sell_cache(s, tmp_path / "m.sell")
    r = read_sell_cache(tmp_path / "m.sell")
    for k in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        assert getattr(r, k).tobytes() == getattr(s, k).tobytes(), k
    x = generate.rhs(m.n_cols)
    assert sb.spmv_sell(r, x).tobytes() == sb.spmv_sell(s, x).tobytes()
    assert sb.spmv_sell(r, x, out_order="original").tobytes() == \
        sb.spmv_sell(s, x, out_order="original").tobytes()


# --- structurally invalid files with a VALID checksum (the
# reference's SellMatrix.__post_init__ rejects them, formats.py:210-251; the
# reader must do the same before any array reaches the device) -------------

def _write_fields(path, **over):
    from types import SimpleNamespace
    g = ref("rand")
    f = {k: g[k] for k in ("cs", "cl", "col", "val", "perm")}
    f.update(n_rows=int(g["n_rows"]), n_cols=int(g["n_cols"]), C=int(g["C"]),
             sigma=int(g["sigma"]), n_rows_padded=int(g["n_rows_padded"]),
             n_chunks=int(g["n_chunks"]), col_permuted=bool(g["col_permuted"]))
    f.update(over)
    write_sell_cache(SimpleNamespace(**f), path)
    return path


@pytest.mark.parametrize("case,match", [
    ("short_col", "col/val length must equal"),
    ("short_val", "col/val length must equal"),
    ("col_out_of_range", "column index out of bounds"),
    ("cl_vs_cs", "cs\\[i\\+1\\] - cs\\[i\\] must equal"),
    ("cs0", "cs\\[0\\] must be 0"),
    ("perm_dup", "perm must be a permutation"),
    ("perm_range", "perm must be a permutation"),
])
def test_structurally_invalid_file_is_rejected(tmp_path, case, match):
    from paper_1307_6209_b200 import StructuralError
    g = ref("rand")
    over = {}
    if case == "short_col":
        over["col"] = g["col"][:-7]
    elif case == "short_val":
        over["val"] = g["val"][:-1]
    elif case == "col_out_of_range":
        c = g["col"].copy()
        c[len(c) // 2] = int(g["n_cols"]) + 3
        over["col"] = c
    elif case == "cl_vs_cs":
        cl = g["cl"].copy()
        cl[0] += 1
        over["cl"] = cl
    elif case == "cs0":
        over["cs"] = g["cs"] + 32
    elif case == "perm_dup":
        p = g["perm"].copy()
        p[1] = p[0]
        over["perm"] = p
    elif case == "perm_range":
        p = g["perm"].copy()
        p[0] = int(g["n_rows"]) + 10
        over["perm"] = p
    path = _write_fields(tmp_path / "bad.sell", **over)
    with pytest.raises(StructuralError, match=match):
        read_sell_cache(path)
