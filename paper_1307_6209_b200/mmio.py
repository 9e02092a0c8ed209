"""Matrix Market ingestion and writing, drop-in for the reference's
``read_matrix_market`` / ``write_matrix_market`` (/root/reference/pkg/src/
sellkit/io.py:192-259), with the text work done natively:

* the body is parsed by ``sellb_mm_parse_body`` (csrc/sellb_mm.cu: all host
  threads, strtod in the C locale -- the same correctly rounded values as
  the reference's np.loadtxt batches, io.py:125-162).  Text outside the fast
  grammar falls back to a NumPy restatement of the reference's reader, so
  every FormatError carries the reference's message and line number;
* canonicalisation runs on the GPU when ``device`` is given
  (``sellb_coo_to_crs``, bit-identical to canonicalize_coo), and
  ``read_matrix_market_sell`` goes file -> device COO -> CRS -> SELL without
  another host pass;
* the writer formats lines with ``sellb_mm_format_body`` -- byte-identical to
  the reference's np.savetxt("%d %d %.17g") output.
"""

import ctypes
import gzip
import os
import warnings

import numpy as np

from . import _lib
from .errors import FormatError
from .formats import COOMatrix, canonicalize_coo, coo_to_crs_device, crs_to_sell_device

_BATCH = 1 << 20            # rows per np.loadtxt batch on the slow path (io.py:18)


# ---------------------------------------------------------------------------
# header (io.py:76-113)
# ---------------------------------------------------------------------------

def _banner_fields(path, banner):
    if not banner or not banner.lstrip().lower().startswith("%%matrixmarket"):
        raise FormatError(f"{path}:1: missing %%MatrixMarket banner")
    words = banner.lower().split()
    if len(words) < 5:
        raise FormatError(f"{path}:1: banner must name object, format, field, symmetry")
    obj, fmt, field, sym = words[1:5]
    if obj != "matrix":
        raise FormatError(f"{path}:1: unsupported object {obj!r} (only 'matrix')")
    if fmt not in ("coordinate", "array"):
        raise FormatError(f"{path}:1: unsupported format {fmt!r}")
    if field == "complex":
        raise FormatError(f"{path}:1: complex matrices are not supported")
    if field not in ("real", "integer", "pattern"):
        raise FormatError(f"{path}:1: unsupported field {field!r}")
    if sym == "hermitian":
        raise FormatError(f"{path}:1: hermitian matrices are not supported")
    if sym not in ("general", "symmetric", "skew-symmetric"):
        raise FormatError(f"{path}:1: unsupported symmetry {sym!r}")
    if fmt == "array" and field == "pattern":
        raise FormatError(f"{path}:1: pattern field is invalid with array format")
    return fmt, field, sym


def _size_fields(path, text, lineno, n_fields):
    """text: the size line (stripped) or None at end of file."""
    if text is None:
        raise FormatError(f"{path}: file ended before the size line")
    parts = text.split()
    if len(parts) != n_fields or not all(p.isdigit() for p in parts):
        raise FormatError(f"{path}:{lineno}: malformed size line {text!r} "
                          f"(expected {n_fields} non-negative integers)")
    return [int(p) for p in parts]


def _is_data(s):
    return bool(s) and not s.startswith("%")


# ---------------------------------------------------------------------------
# failure-path line location (io.py:32-73), by re-reading the text
# ---------------------------------------------------------------------------

def _text_lines(path):
    if str(path).endswith(".gz"):
        return gzip.open(path, "rt")
    return open(path, "r")


def _data_line_number(path, index):
    """Line number of data line `index` (0 = the size line)."""
    seen = -1
    with _text_lines(path) as fh:
        for lineno, line in enumerate(fh, 1):
            if lineno > 1 and _is_data(line.strip()):
                seen += 1
                if seen == index:
                    return lineno
    return None


def _first_bad_line(path, width):
    seen = -1
    with _text_lines(path) as fh:
        for lineno, line in enumerate(fh, 1):
            s = line.strip()
            if lineno == 1 or not _is_data(s):
                continue
            seen += 1
            if seen == 0:
                continue
            words = s.split()
            if len(words) != width:
                return lineno, f"expected {width} values, found {len(words)}"
            try:
                for w in words:
                    float(w)
            except ValueError:
                return lineno, f"unparseable value in {s!r}"
    return None, "malformed entry"


def _line_count(path):
    with _text_lines(path) as fh:
        return sum(1 for _ in fh)


def _malformed(path, width, cause=None):
    lineno, why = _first_bad_line(path, width)
    where = f":{lineno}" if lineno else ""
    err = FormatError(f"{path}{where}: {why}")
    if cause is not None:
        raise err from cause
    raise err


# ---------------------------------------------------------------------------
# body: native fast path, NumPy slow path
# ---------------------------------------------------------------------------

def _slow_read(path, n_fields, width, expected):
    """The reference's reader restated on NumPy (io.py:116-162): header
    re-read in text mode, body in np.loadtxt batches."""
    with _text_lines(path) as fh:
        fh.readline()
        lineno = 1
        while True:
            line = fh.readline()
            if not line:
                break
            lineno += 1
            if _is_data(line.strip()):
                break
        blocks, total = [], 0
        while True:
            try:
                with warnings.catch_warnings():
                    warnings.simplefilter("ignore", UserWarning)
                    blk = np.loadtxt(fh, dtype=np.float64, comments="%", max_rows=_BATCH,
                                     ndmin=2)
            except ValueError as exc:
                _malformed(path, width, exc)
            if blk.size == 0:
                break
            if blk.shape[1] != width:
                _malformed(path, width)
            total += len(blk)
            if total > expected:
                ln = _data_line_number(path, expected + 1)
                raise FormatError(f"{path}:{ln}: more entries than the declared {expected}")
            blocks.append(blk)
    if total < expected:
        raise FormatError(f"{path}:{_line_count(path)}: file ended after {total} of "
                          f"{expected} declared entries")
    return np.concatenate(blocks, axis=0) if blocks else np.zeros((0, width))


def _split_header(raw):
    """(banner, size_line_text, size_lineno, body_offset) from the raw
    bytes, or None when the header needs the text-mode reader (a lone CR,
    undecodable bytes)."""
    pos, lineno, banner, size = 0, 0, None, None
    n = len(raw)
    while pos < n or banner is None:
        nl = raw.find(b"\n", pos)
        end = n if nl < 0 else nl + 1
        line = raw[pos:end]
        body = line[:-1] if line.endswith(b"\n") else line
        if body.endswith(b"\r"):
            body = body[:-1]
        if b"\r" in body:
            return None
        try:
            text = body.decode()
        except UnicodeDecodeError:
            return None
        lineno += 1
        pos = end
        if banner is None:
            banner = text
            if pos >= n:
                return banner, None, lineno, pos
            continue
        if _is_data(text.strip()):
            size = text.strip()
            return banner, size, lineno, pos
        if pos >= n:
            break
    return banner, size, lineno, pos


def _read_raw(path):
    if str(path).endswith(".gz"):
        with gzip.open(path, "rb") as fh:
            return fh.read()
    with open(path, "rb") as fh:
        return fh.read()


def _parse_body(raw, off, width, expected):
    """Fast path: the body bytes -> (n, width) float64, or None to fall back."""
    lib = _lib.load()
    out = np.empty(max(expected, 1) * width, dtype=np.float64)
    cnt = ctypes.c_int64()
    buf = ctypes.c_char_p(raw)
    base = ctypes.cast(buf, ctypes.c_void_p).value
    rc = lib.sellb_mm_parse_body(base + off, len(raw) - off, width, expected,
                                 out.ctypes.data, ctypes.byref(cnt), 0)
    if rc != 0:
        return None
    n = cnt.value
    if n < expected:
        return None                      # short file: the slow path reports it
    return out[:n * width].reshape(n, width)


def _read_triplets(path):
    """(n_rows, n_cols, rows, cols, vals, fmt, symmetry) before expansion."""
    raw = _read_raw(path)
    head = _split_header(raw)
    if head is None:
        # header needs universal-newline text mode: mirror it exactly
        with _text_lines(path) as fh:
            banner = fh.readline()
            fmt, field, sym = _banner_fields(path, banner)
            lineno, size = 1, None
            while True:
                line = fh.readline()
                if not line:
                    break
                lineno += 1
                if _is_data(line.strip()):
                    size = line.strip()
                    break
        off = None
    else:
        banner, size, lineno, off = head
        fmt, field, sym = _banner_fields(path, banner)
    if fmt == "coordinate":
        n_rows, n_cols, nnz = _size_fields(path, size, lineno, 3)
        width, expected = (2 if field == "pattern" else 3), nnz
    else:
        n_rows, n_cols = _size_fields(path, size, lineno, 2)
        if sym != "general" and n_rows != n_cols:
            raise FormatError(f"{path}: {sym} array storage requires a square matrix")
        skip = 1 if sym == "skew-symmetric" else 0
        d = n_rows - skip
        width, expected = 1, (n_rows * n_cols if sym == "general" else d * (d + 1) // 2)
    body = _parse_body(raw, off, width, expected) if off is not None else None
    del raw
    if body is None:
        body = _slow_read(path, 3 if fmt == "coordinate" else 2, width, expected)
    if fmt == "coordinate":
        for k, (axis, upper) in enumerate((("row", n_rows), ("column", n_cols))):
            idx = body[:, k]
            with np.errstate(invalid="ignore"):
                bad = (idx < 1) | (idx > upper) | (idx != np.floor(idx))
            if bad.any():
                i = int(np.flatnonzero(bad)[0])
                ln = _data_line_number(path, i + 1)
                raise FormatError(f"{path}:{ln}: {axis} index {idx[i]:g} out of range "
                                  f"1..{upper}")
        rows = body[:, 0].astype(np.int64) - 1
        cols = body[:, 1].astype(np.int64) - 1
        vals = body[:, 2].copy() if width == 3 else np.ones(len(body))
    else:
        rows, cols = _array_positions(n_rows, n_cols, sym, expected)
        vals = body[:, 0].copy()
        nz = vals != 0.0                       # dense storage: zeros are not entries
        rows, cols, vals = rows[nz], cols[nz], vals[nz]
    return n_rows, n_cols, rows, cols, vals, fmt, sym


def _array_positions(n_rows, n_cols, sym, count):
    """Column-major storage positions -> (row, col) (io.py:176-189)."""
    k = np.arange(count, dtype=np.int64)
    if sym == "general":
        return (k % n_rows, k // n_rows) if n_rows else (k, k)
    skip = 1 if sym == "skew-symmetric" else 0
    per_col = np.maximum(n_rows - skip - np.arange(n_cols, dtype=np.int64), 0)
    first = np.zeros(n_cols + 1, dtype=np.int64)
    np.cumsum(per_col, out=first[1:])
    c = np.searchsorted(first, k, side="right") - 1
    return c + skip + (k - first[c]), c


def _expanded(path, rows, cols, vals, fmt, sym):
    if sym == "general":
        return rows, cols, vals
    if sym == "skew-symmetric":
        diag = rows == cols
        if diag.any():
            i = int(np.flatnonzero(diag)[0])
            ln = _data_line_number(path, i + 1) if fmt == "coordinate" else None
            where = f":{ln}" if ln else ""
            raise FormatError(f"{path}{where}: skew-symmetric matrices cannot have "
                              "diagonal entries")
    mirror = rows != cols
    sign = -1.0 if sym == "skew-symmetric" else 1.0
    return (np.concatenate([rows, cols[mirror]]), np.concatenate([cols, rows[mirror]]),
            np.concatenate([vals, sign * vals[mirror]]))


def read_matrix_market(path, *, device=None):
    """Parse a Matrix Market file (.mtx / .mtx.gz) into canonical triplet form
    (io.py:192-240): symmetric / skew-symmetric storage expanded, pattern
    entries 1.0, 1-based indices made 0-based, duplicates summed.
    ``device=k`` canonicalises on GPU k (same result)."""
    path = os.fspath(path)
    n_rows, n_cols, rows, cols, vals, fmt, sym = _read_triplets(path)
    rows, cols, vals = _expanded(path, rows, cols, vals, fmt, sym)
    coo = COOMatrix(n_rows, n_cols, rows, cols, vals)
    if device is None:
        return canonicalize_coo(coo)
    d = coo_to_crs_device(coo, device=device)
    rpt = d.rpt.cpu().numpy()
    r = np.repeat(np.arange(n_rows, dtype=np.int64), np.diff(rpt))
    return COOMatrix(n_rows, n_cols, r, d.col.cpu().numpy().astype(np.int64),
                     d.val.cpu().numpy())


def read_matrix_market_sell(path, C, sigma, align_bytes=1, permute_cols=False, *, device=0,
                            stream=None):
    """File -> SELL-C-sigma: native parse, then COO -> CRS -> SELL on the GPU
    (the reference's crs_to_sell(coo_to_crs(read_matrix_market(path)))."""
    path = os.fspath(path)
    n_rows, n_cols, rows, cols, vals, fmt, sym = _read_triplets(path)
    rows, cols, vals = _expanded(path, rows, cols, vals, fmt, sym)
    d = coo_to_crs_device(COOMatrix(n_rows, n_cols, rows, cols, vals), device=device,
                          stream=stream)
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device).cuda_stream
    return crs_to_sell_device(d.rpt, d.col, d.val, n_rows, n_cols, C, sigma, align_bytes,
                              permute_cols, device=device, stream=stream)


def write_matrix_market(m, path, comment=None):
    """General real coordinate file of the canonical triplets (io.py:243-259);
    the same bytes as the reference's writer."""
    m = canonicalize_coo(m)
    path = os.fspath(path)
    lib = _lib.load()
    opener = (lambda: gzip.open(path, "wb")) if path.endswith(".gz") else \
        (lambda: open(path, "wb"))
    with opener() as fh:
        fh.write(b"%%MatrixMarket matrix coordinate real general\n")
        if comment:
            fh.write(f"%{comment}\n".encode())
        fh.write(f"{m.n_rows} {m.n_cols} {m.nnz}\n".encode())
        used = ctypes.c_int64()
        for a in range(0, m.nnz, _BATCH):
            b = min(a + _BATCH, m.nnz)
            buf = ctypes.create_string_buffer((b - a) * 64 + 64)
            _lib.check(lib.sellb_mm_format_body(
                m.rows[a:b].ctypes.data, m.cols[a:b].ctypes.data, m.vals[a:b].ctypes.data,
                b - a, ctypes.addressof(buf), len(buf), ctypes.byref(used), 0))
            fh.write(buf.raw[:used.value])
