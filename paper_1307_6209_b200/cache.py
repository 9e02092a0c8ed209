"""Binary ``.sell`` cache files straight to and from device memory (SURVEY.md
§8(f) item 2) -- the on-disk format of the reference's
``write_sell_cache`` / ``read_sell_cache`` (/root/reference/pkg/src/sellkit/
io.py:243-382, SPEC.md "External Interfaces"), byte-compatible both ways:

    "SELL" | u16 version=1 | u16 flags (bit0: col_permuted)
    | u64 n_rows, n_cols, C, sigma, n_rows_padded, n_chunks
    | (u64 count, data) for cs u64, cl u32, col u32, val f64, perm u32
    | u32 CRC-32 of everything before it            (all little-endian)

Reading validates magic, version, array lengths, truncation and the CRC with
the reference's FormatError messages, then uploads the arrays once and
rebuilds ``row_lengths`` ON THE DEVICE with the reference's rule
(trailing run of value-0.0 / column-0 slots, io.py:308-321; sellb_infer_row_
lengths).  Like the reference, a row whose last stored entries are explicit
zeros in column 0 reads back shorter -- harmless for y (those slots add
0*x[0] either way) but visible in ``row_lengths`` / ``nnz``.
"""

import ctypes
import os
import struct
import zlib

import numpy as np

from . import _lib
from .errors import FormatError
from .formats import SellMatrix, validate_sell_arrays

MAGIC = b"SELL"
VERSION = 1
FLAG_COL_PERMUTED = 1

_ARRAYS = (("cs", "<u8", np.int64), ("cl", "<u4", np.int32), ("col", "<u4", np.int32),
           ("val", "<f8", np.float64), ("perm", "<u4", np.int32))


def write_sell_cache(m, path):
    """Write a SELL-C-sigma matrix (device-resident or host-built) in the
    reference's cache layout; values are stored as f64 (the format's type)."""
    path = os.fspath(path)
    flags = FLAG_COL_PERMUTED if m.col_permuted else 0
    crc = 0
    with open(path, "wb") as fh:
        def put(data):
            nonlocal crc
            fh.write(data)
            crc = zlib.crc32(data, crc)
        put(struct.pack("<4sHH", MAGIC, VERSION, flags))
        put(struct.pack("<6Q", m.n_rows, m.n_cols, m.C, m.sigma, m.n_rows_padded,
                        m.n_chunks))
        for name, disk, _ in _ARRAYS:
            arr = np.ascontiguousarray(getattr(m, name), dtype=disk)
            put(struct.pack("<Q", len(arr)))
            put(memoryview(arr).cast("B"))
        fh.write(struct.pack("<I", crc))


def read_sell_cache(path, device=0):
    """Read a cache file into a device-resident SellMatrix, verifying it."""
    path = os.fspath(path)
    with open(path, "rb") as fh:
        blob = fh.read()
    pos = 0
    crc = 0

    def take(n):
        nonlocal pos, crc
        if pos + n > len(blob):
            raise FormatError(f"{path}: truncated file")
        view = memoryview(blob)[pos:pos + n]
        crc = zlib.crc32(view, crc)
        pos += n
        return view

    magic, version, flags = struct.unpack("<4sHH", take(8))
    if magic != MAGIC:
        raise FormatError(f"{path}: not a chunked-matrix cache file")
    if version != VERSION:
        raise FormatError(f"{path}: cache version {version} not supported "
                          f"(expected {VERSION})")
    n_rows, n_cols, C, sigma, n_pad, n_chunks = struct.unpack("<6Q", take(48))
    want = {"cs": n_chunks + 1, "cl": n_chunks, "col": None, "val": None, "perm": n_rows}
    arrays = {}
    for name, disk, host in _ARRAYS:
        (count,) = struct.unpack("<Q", take(8))
        if want[name] is not None and count != want[name]:
            raise FormatError(f"{path}: array {name} has {count} elements, "
                              f"expected {want[name]}")
        raw = take(count * np.dtype(disk).itemsize)
        arrays[name] = np.frombuffer(raw, dtype=disk).view(host)
    if pos + 4 > len(blob):
        raise FormatError(f"{path}: truncated file")
    (stored,) = struct.unpack("<I", blob[pos:pos + 4])
    if stored != crc:
        raise FormatError(f"{path}: checksum failure (corrupted cache)")

    # the reference builds a SellMatrix from the arrays, whose __post_init__
    # rejects a structurally invalid file (valid CRC, inconsistent arrays)
    # with StructuralError before anything indexes them (formats.py:210-251)
    h = dict(arrays, row_lengths=None)
    h["perm"] = arrays["perm"].astype(np.int64) if len(arrays["perm"]) else arrays["perm"]
    validate_sell_arrays(int(n_rows), int(n_cols), int(C), int(sigma), int(n_pad),
                         int(n_chunks), h)
    lib = _lib.require_device()
    out = ctypes.c_void_p()
    _lib.check(lib.sellb_import(
        _lib.ptr(arrays["cs"]), _lib.ptr(arrays["cl"]), _lib.ptr(arrays["col"]),
        _lib.ptr(arrays["val"]), _lib.ptr(arrays["perm"]), None, _lib.SELLB_F64,
        int(n_rows), int(n_cols), int(C), int(sigma), int(n_chunks), len(arrays["val"]),
        int(bool(flags & FLAG_COL_PERMUTED)), int(device), None, 0, ctypes.byref(out)))
    try:
        _lib.check(lib.sellb_infer_row_lengths(out.value, None))
    except Exception:
        lib.sellb_free(out.value)
        raise
    s = SellMatrix._adopt(out.value, int(sigma))
    if s.n_rows_padded != n_pad:
        raise FormatError(f"{path}: n_rows_padded {n_pad} inconsistent with n_chunks * C")
    return s
