"""Sparse containers and the SELL-C-sigma build, drop-in for the reference
``sellkit.formats`` (/root/reference/pkg/src/sellkit/formats.py).

Host side:
    COOMatrix, CRSMatrix, canonicalize_coo, coo_to_crs, crs_to_coo -- the
    input containers (NumPy, validated like formats.py:35-180).
Device side:
    crs_to_sell -- the SELL-C-sigma build runs on the GPU through
    ``sellb_build_from_crs`` (csrc/sellb_build.cu).  The returned SellMatrix is
    device-resident; its NumPy array fields (cs, cl, col, val, perm,
    row_lengths) are exported lazily on first access and are bit-identical to
    the reference's (formats.py:295-393).

Conventions kept from the reference: values float64 (float32 on request),
column indices int32, offsets int64, ``perm`` maps original row -> stored
row, containers are immutable after construction.
"""

import ctypes
import weakref

import numpy as np

from . import _lib
from .errors import DimensionError, ParameterError, StructuralError

VALUE_DTYPE = np.float64
INDEX_DTYPE = np.int32
OFFSET_DTYPE = np.int64
MAX_DIM = 2 ** 31          # 4-byte index semantics (formats.py:22-23)


def _check_dims(n_rows, n_cols):
    if n_rows < 0 or n_cols < 0:
        raise StructuralError(f"negative matrix dimension ({n_rows}x{n_cols})")
    if max(n_rows, n_cols) >= MAX_DIM:
        raise StructuralError(
            f"matrix dimension {max(n_rows, n_cols)} exceeds 4-byte index range")


# ---------------------------------------------------------------------------
# COO / CRS (host input containers; formats.py:35-180)
# ---------------------------------------------------------------------------

class COOMatrix:
    """Triplet matrix, possibly unsorted with duplicates (formats.py:35-86)."""

    def __init__(self, n_rows, n_cols, rows, cols, vals):
        _check_dims(n_rows, n_cols)
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.rows = np.ascontiguousarray(rows, dtype=OFFSET_DTYPE)
        self.cols = np.ascontiguousarray(cols, dtype=OFFSET_DTYPE)
        self.vals = np.ascontiguousarray(vals, dtype=VALUE_DTYPE)
        if not self.rows.ndim == self.cols.ndim == self.vals.ndim == 1:
            raise StructuralError("entry arrays must be one-dimensional")
        if not len(self.rows) == len(self.cols) == len(self.vals):
            raise StructuralError("entry arrays must have equal length")
        if len(self.rows):
            bad_r = (self.rows < 0) | (self.rows >= self.n_rows)
            if bad_r.any():
                raise StructuralError(
                    f"row index {int(self.rows[bad_r][0])} out of bounds for "
                    f"{self.n_rows} rows")
            bad_c = (self.cols < 0) | (self.cols >= self.n_cols)
            if bad_c.any():
                raise StructuralError(
                    f"column index {int(self.cols[bad_c][0])} out of bounds for "
                    f"{self.n_cols} columns")

    @property
    def nnz(self):
        return len(self.vals)

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def is_canonical(self):
        if self.nnz < 2:
            return True
        dr = np.diff(self.rows)
        return bool(np.all((dr > 0) | ((dr == 0) & (np.diff(self.cols) > 0))))


def canonicalize_coo(m):
    """Row-major sort, duplicates summed, explicit zeros kept
    (formats.py:89-108)."""
    if m.is_canonical():
        return m
    key_order = np.lexsort((m.cols, m.rows))
    r, c, v = m.rows[key_order], m.cols[key_order], m.vals[key_order]
    if len(r) > 1:
        new = np.ones(len(r), dtype=bool)
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        if not new.all():
            first = np.flatnonzero(new)
            v = np.add.reduceat(v, first)
            r, c = r[first], c[first]
    return COOMatrix(m.n_rows, m.n_cols, r, c, v)


class CRSMatrix:
    """Row-pointer matrix: rpt int64[n+1], col int32[nnz], val f64[nnz];
    strictly increasing columns within a row (formats.py:111-166)."""

    def __init__(self, n_rows, n_cols, rpt, col, val):
        _check_dims(n_rows, n_cols)
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.rpt = np.ascontiguousarray(rpt, dtype=OFFSET_DTYPE)
        self.col = np.ascontiguousarray(col, dtype=INDEX_DTYPE)
        val = np.asarray(val)
        self.val = np.ascontiguousarray(
            val, dtype=np.float32 if val.dtype == np.float32 else VALUE_DTYPE)
        if len(self.rpt) != self.n_rows + 1:
            raise StructuralError(f"rpt has length {len(self.rpt)}, expected "
                                  f"n_rows+1 = {self.n_rows + 1}")
        if self.n_rows and self.rpt[0] != 0:
            raise StructuralError("rpt[0] must be 0")
        if self.rpt[-1] != len(self.col):
            raise StructuralError("rpt[-1] must equal the number of stored entries")
        if len(self.col) != len(self.val):
            raise StructuralError("col and val must have equal length")
        lens = np.diff(self.rpt)
        if len(lens) and lens.min() < 0:
            raise StructuralError("rpt must be non-decreasing")
        nnz = len(self.col)
        if nnz:
            if self.col.min() < 0 or self.col.max() >= self.n_cols:
                raise StructuralError("column index out of bounds")
            if nnz > 1:
                step_ok = np.diff(self.col) > 0
                # a new row may restart the column sequence
                boundary = self.rpt[1:-1]
                boundary = boundary[(boundary > 0) & (boundary < nnz)] - 1
                step_ok[boundary] = True
                if not step_ok.all():
                    raise StructuralError(
                        "column indices must be strictly increasing within each row")

    @property
    def nnz(self):
        return len(self.val)

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def row_lengths(self):
        return np.diff(self.rpt)


def coo_to_crs(m, *, device=None, stream=None):
    """formats.py:169-175.

    ``device=None`` keeps the reference's host conversion; ``device=k`` runs
    the canonicalisation on GPU k (``sellb_coo_to_crs``, csrc/sellb_coo.cu)
    and returns the same CRSMatrix bit for bit (duplicate sums included)."""
    if device is not None:
        lib = _lib.require_device()
        rpt = np.zeros(m.n_rows + 1, dtype=OFFSET_DTYPE)
        col = np.empty(m.nnz, dtype=INDEX_DTYPE)
        val = np.empty(m.nnz, dtype=VALUE_DTYPE)
        nnz = ctypes.c_int64()
        _lib.check(lib.sellb_coo_to_crs(
            _lib.ptr(m.rows), _lib.ptr(m.cols), _lib.ptr(m.vals), m.nnz, m.n_rows,
            m.n_cols, _lib.ptr(rpt), _lib.ptr(col), _lib.ptr(val), ctypes.byref(nnz),
            int(device), stream, 0))
        n = nnz.value
        return CRSMatrix(m.n_rows, m.n_cols, rpt, col[:n], val[:n])
    m = canonicalize_coo(m)
    rpt = np.zeros(m.n_rows + 1, dtype=OFFSET_DTYPE)
    np.cumsum(np.bincount(m.rows, minlength=m.n_rows), out=rpt[1:])
    return CRSMatrix(m.n_rows, m.n_cols, rpt, m.cols.astype(INDEX_DTYPE), m.vals)


class DeviceCRS:
    """Canonical CRS held in CUDA tensors (rpt int64, col int32, val f64) --
    the device-side input of ``crs_to_sell_device``; ``to_host()`` gives the
    CRSMatrix."""

    def __init__(self, n_rows, n_cols, rpt, col, val):
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.rpt, self.col, self.val = rpt, col, val

    @property
    def nnz(self):
        return int(self.col.numel())

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    def to_host(self):
        return CRSMatrix(self.n_rows, self.n_cols, self.rpt.cpu().numpy(),
                         self.col.cpu().numpy(), self.val.cpu().numpy())


def coo_to_crs_device(m, *, device=0, stream=None):
    """COO (a COOMatrix, or a tuple ``(n_rows, n_cols, rows, cols, vals)`` of
    CUDA tensors int64/int64/f64) -> DeviceCRS, canonicalised on the GPU
    (formats.py:89-108,169-175; bit-identical).  Runs on ``stream`` (default:
    torch's current stream of ``device``)."""
    import torch
    lib = _lib.require_device()
    dev = torch.device("cuda", device)
    if isinstance(m, COOMatrix):
        n_rows, n_cols = m.n_rows, m.n_cols
        rows = torch.from_numpy(m.rows).to(dev)
        cols = torch.from_numpy(m.cols).to(dev)
        vals = torch.from_numpy(m.vals).to(dev)
    else:
        n_rows, n_cols, rows, cols, vals = m
        _check_dims(n_rows, n_cols)
        if not (rows.dtype == cols.dtype == torch.int64 and vals.dtype == torch.float64):
            raise ParameterError("rows/cols must be int64 and vals float64 tensors")
        if not rows.numel() == cols.numel() == vals.numel():
            raise StructuralError("entry arrays must have equal length")
        rows, cols, vals = rows.contiguous(), cols.contiguous(), vals.contiguous()
    nnz_in = int(vals.numel())
    rpt = torch.empty(int(n_rows) + 1, dtype=torch.int64, device=dev)
    col = torch.empty(nnz_in, dtype=torch.int32, device=dev)
    val = torch.empty(nnz_in, dtype=torch.float64, device=dev)
    if stream is None:
        stream = torch.cuda.current_stream(dev).cuda_stream
    nnz = ctypes.c_int64()
    _lib.check(lib.sellb_coo_to_crs(
        rows.data_ptr(), cols.data_ptr(), vals.data_ptr(), nnz_in, int(n_rows), int(n_cols),
        rpt.data_ptr(), col.data_ptr(), val.data_ptr(), ctypes.byref(nnz), int(device),
        stream, 1))
    n = nnz.value
    return DeviceCRS(n_rows, n_cols, rpt, col[:n], val[:n])


def coo_to_sell(m, C, sigma, align_bytes=1, permute_cols=False, *, device=0, stream=None):
    """COO -> canonical CRS -> SELL-C-sigma without leaving the GPU: the
    reference's ``crs_to_sell(coo_to_crs(m), ...)`` (formats.py:169-175,
    295-393) in two device passes; identical SellMatrix."""
    d = coo_to_crs_device(m, device=device, stream=stream)
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(device).cuda_stream
    return crs_to_sell_device(d.rpt, d.col, d.val, d.n_rows, d.n_cols, C, sigma,
                              align_bytes, permute_cols, device=device, stream=stream)


def crs_to_coo(m):
    """formats.py:178-180."""
    rows = np.repeat(np.arange(m.n_rows, dtype=OFFSET_DTYPE), m.row_lengths())
    return COOMatrix(m.n_rows, m.n_cols, rows, m.col.astype(OFFSET_DTYPE),
                     m.val.astype(VALUE_DTYPE))


# ---------------------------------------------------------------------------
# SELL-C-sigma (device-resident)
# ---------------------------------------------------------------------------

_ARRAYS = ("cs", "cl", "col", "val", "perm", "row_lengths")


def validate_sell_arrays(n_rows, n_cols, C, sigma, n_rows_padded, n_chunks, h):
    """The reference's SellMatrix.__post_init__ invariants (formats.py:210-251)
    on host arrays h = {cs, cl, col, val, perm, row_lengths}; row_lengths may
    be None (a .sell cache: rebuilt on the device afterwards, within [0, cl]
    by construction).  Same exception classes and messages."""
    if C < 1:
        raise ParameterError(f"chunk height C must be >= 1, got {C}")
    if sigma < 1:
        raise ParameterError(f"sigma must be >= 1, got {sigma}")
    if n_chunks * C != n_rows_padded:
        raise StructuralError("n_rows_padded must equal n_chunks * C")
    if not n_rows <= n_rows_padded < n_rows + C:
        if not (n_rows == 0 and n_rows_padded == 0):
            raise StructuralError("n_rows_padded must be n_rows rounded up to C")
    cs, cl = h["cs"], h["cl"]
    if len(cs) != n_chunks + 1 or len(cl) != n_chunks:
        raise StructuralError("cs/cl length mismatch with n_chunks")
    if len(cs) and cs[0] != 0:
        raise StructuralError("cs[0] must be 0")
    if np.any(np.diff(cs) != C * cl.astype(OFFSET_DTYPE)):
        raise StructuralError("cs[i+1] - cs[i] must equal C * cl[i]")
    total = int(cs[-1]) if len(cs) else 0
    if len(h["col"]) != total or len(h["val"]) != total:
        raise StructuralError("col/val length must equal cs[n_chunks]")
    perm = h["perm"]
    if len(perm) != n_rows:
        raise StructuralError("perm must have length n_rows")
    if n_rows:
        if perm.min() < 0 or perm.max() >= n_rows or \
                np.any(np.bincount(perm, minlength=n_rows) != 1):
            raise StructuralError("perm must be a permutation of 0..n_rows-1")
    rl = h.get("row_lengths")
    if rl is not None:
        if len(rl) != n_rows_padded:
            raise StructuralError("row_lengths must have length n_rows_padded")
        if n_rows_padded:
            cap = np.repeat(cl, C)
            if np.any(rl > cap) or np.any(rl < 0):
                raise StructuralError("row length outside [0, cl] for its chunk")
            if np.any(rl[n_rows:] != 0):
                raise StructuralError("padding rows must have length 0")
    if total and n_cols == 0:
        raise StructuralError("stored slots require n_cols >= 1")
    if total and (h["col"].min() < 0 or h["col"].max() >= n_cols):
        raise StructuralError("column index out of bounds")


class SellMatrix:
    """Chunked, sorted-row sparse matrix living in GPU memory.

    Same fields and invariants as the reference SellMatrix
    (formats.py:183-271): element (stored row p, slot j) at
    ``cs[p // C] + j*C + p % C``; padding slots hold 0.0 / column 0; stored
    rows [n_rows, n_rows_padded) are empty padding rows.

    Built by ``crs_to_sell`` (device build) or constructed from host arrays
    exactly like the reference dataclass (validated on the host, uploaded on
    first use).  Array attributes are NumPy views exported on first access.
    """

    def __init__(self, n_rows, n_cols, C, sigma, n_rows_padded, n_chunks, cs,
                 cl, col, val, perm, row_lengths, col_permuted=False, *,
                 device=0):
        _check_dims(n_rows, n_cols)
        self.n_rows, self.n_cols = int(n_rows), int(n_cols)
        self.C, self.sigma = int(C), int(sigma)
        self.n_rows_padded, self.n_chunks = int(n_rows_padded), int(n_chunks)
        self.col_permuted = bool(col_permuted)
        self.device = int(device)
        self._handle = None
        self._finalizer = None
        self._nnz = None
        self._slots = None
        val = np.asarray(val)
        vdt = np.float32 if val.dtype == np.float32 else VALUE_DTYPE
        self._host = {
            "cs": np.ascontiguousarray(cs, dtype=OFFSET_DTYPE),
            "cl": np.ascontiguousarray(cl, dtype=INDEX_DTYPE),
            "col": np.ascontiguousarray(col, dtype=INDEX_DTYPE),
            "val": np.ascontiguousarray(val, dtype=vdt),
            "perm": np.ascontiguousarray(perm, dtype=INDEX_DTYPE),
            "row_lengths": np.ascontiguousarray(row_lengths, dtype=INDEX_DTYPE),
        }
        self.dtype = np.dtype(vdt)
        self._inv_perm = None
        self._validate_host()

    # -- construction from a device handle ---------------------------------
    @classmethod
    def _adopt(cls, handle, sigma):
        self = cls.__new__(cls)
        info = _lib.Info()
        _lib.check(_lib.load().sellb_info(handle, ctypes.byref(info)))
        self.n_rows, self.n_cols = int(info.n_rows), int(info.n_cols)
        self.C, self.sigma = int(info.C), int(sigma)
        self.n_rows_padded, self.n_chunks = int(info.n_rows_padded), int(info.n_chunks)
        self.col_permuted = bool(info.col_permuted)
        self.device = int(info.device)
        self.dtype = np.dtype(np.float32 if info.dtype == _lib.SELLB_F32 else np.float64)
        self._nnz = int(info.nnz)
        self._slots = int(info.slots)
        self._host = dict.fromkeys(_ARRAYS)
        self._inv_perm = None
        self._attach(handle)
        return self

    def _attach(self, handle):
        self._handle = handle
        self._finalizer = weakref.finalize(self, _free_handle, handle)

    def _validate_host(self):
        """The reference's __post_init__ invariants (formats.py:210-251)."""
        validate_sell_arrays(self.n_rows, self.n_cols, self.C, self.sigma,
                             self.n_rows_padded, self.n_chunks, self._host)

    # -- device side -----------------------------------------------------------
    @property
    def handle(self):
        """The ``sellb_mat*`` (uploads host-constructed matrices on first use)."""
        if self._handle is None:
            h = self._host
            if any(h.get(k) is None for k in _ARRAYS):
                from .errors import ResourceError
                raise ResourceError("the matrix's device copy was freed")
            lib = _lib.require_device()
            out = ctypes.c_void_p()
            dt = _lib.SELLB_F32 if self.dtype == np.float32 else _lib.SELLB_F64
            _lib.check(lib.sellb_import(
                _lib.ptr(h["cs"]), _lib.ptr(h["cl"]), _lib.ptr(h["col"]),
                _lib.ptr(h["val"]), _lib.ptr(h["perm"]), _lib.ptr(h["row_lengths"]),
                dt, self.n_rows, self.n_cols, self.C, self.sigma, self.n_chunks,
                len(h["val"]), int(self.col_permuted), self.device, None, 0,
                ctypes.byref(out)))
            self._attach(out.value)
        return self._handle

    def info(self):
        info = _lib.Info()
        _lib.check(_lib.load().sellb_info(self.handle, ctypes.byref(info)))
        return info

    def device_arrays(self):
        """Raw device pointers (ints) of cs, cl, col, val, perm, order,
        row_lengths."""
        d = _lib.DevArrays()
        _lib.check(_lib.load().sellb_device_arrays(self.handle, ctypes.byref(d)))
        return {name: getattr(d, name) for name, _ in d._fields_}

    def streamed_bytes(self):
        """(matrix bytes at 32-byte sectors, at 64-byte granularity, extra
        row_lengths bytes) the SpMV streams as configured (sellb_streamed_bytes)."""
        a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.require_device().sellb_streamed_bytes(
            self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c), None))
        return a.value, b.value, c.value

    def long_rows_info(self):
        """How the long rows are handled: {"n_long", "n_groups", "n_rest",
        "side_entries"} (sellb_long_info)."""
        vals = [ctypes.c_int64() for _ in range(4)]
        _lib.check(_lib.require_device().sellb_long_info(self.handle,
                                                         *[ctypes.byref(v) for v in vals]))
        return dict(zip(("n_long", "n_groups", "n_rest", "side_entries"),
                        (v.value for v in vals)))

    def sector_occupancy(self):
        """(beta_eff, val_sectors, col_sectors): occupancy counted in the
        32-byte sectors the pad-skipping kernel touches."""
        be = ctypes.c_double()
        vs, cs = ctypes.c_int64(), ctypes.c_int64()
        _lib.check(_lib.load().sellb_sector_occupancy(self.handle, ctypes.byref(be),
                                                      ctypes.byref(vs), ctypes.byref(cs),
                                                      None))
        return float(be.value), int(vs.value), int(cs.value)

    def export_range(self, c0, c1):
        """Host copies of chunks [c0, c1): cs (rebased), cl, col, val and
        row_lengths -- block-wise parity without exporting the whole matrix."""
        info = self.info()
        c0, c1 = int(c0), int(c1)
        lib = _lib.load()
        cs = np.empty(c1 - c0 + 1, OFFSET_DTYPE)
        _lib.check(lib.sellb_export_range(self.handle, c0, c1, _lib.ptr(cs), None, None,
                                          None, None))
        slots = int(cs[-1])
        out = {"cs": cs, "cl": np.empty(c1 - c0, INDEX_DTYPE),
               "col": np.empty(slots, INDEX_DTYPE), "val": np.empty(slots, self.dtype),
               "row_lengths": np.empty((c1 - c0) * int(info.C), INDEX_DTYPE)}
        _lib.check(lib.sellb_export_range(self.handle, c0, c1, None, _lib.ptr(out["cl"]),
                                          _lib.ptr(out["col"]), _lib.ptr(out["val"]),
                                          _lib.ptr(out["row_lengths"])))
        return out

    @property
    def variant(self):
        return {1: "pad_skip", 2: "pad_incl"}.get(self.info().variant, "auto")

    @property
    def packed(self):
        """Whether the SpMV streams the packed chunk copy (pad-heavy C = 32
        layouts; the exported SELL arrays are unchanged)."""
        return bool(self.info().packed)

    def set_packed(self, mode):
        """True builds the packed chunk copy, False drops it, None lets the
        build's cost model decide (sellb_set_packed)."""
        code = -1 if mode is None else (1 if mode else 0)
        _lib.check(_lib.load().sellb_set_packed(self.handle, code))

    @property
    def shadow(self):
        """Whether whole-matrix SpMVs run on a SELL-32 shadow layout of the
        same rows (irregular layouts; the exported arrays are unchanged)."""
        return bool(self.info().shadow)

    @property
    def shadow_sigma(self):
        """The shadow layout's sigma (n_rows: SELL-32-N, x in L2; 512 for
        larger x), 0 without a shadow."""
        return int(self.info().shadow)

    def set_shadow(self, mode):
        """True builds the shadow layout, False drops it, None lets the
        build's cost model decide (sellb_set_shadow)."""
        code = -1 if mode is None else (1 if mode else 0)
        _lib.check(_lib.load().sellb_set_shadow(self.handle, code))

    def set_variant(self, name):
        code = {"auto": _lib.VARIANT_AUTO, "pad_skip": _lib.VARIANT_PAD_SKIP,
                "pad_incl": _lib.VARIANT_PAD_INCL}.get(name)
        if code is None:
            raise ParameterError(f"unknown kernel variant {name!r}")
        _lib.check(_lib.load().sellb_set_variant(self.handle, code))

    def free(self):
        """Release the device copy now (host arrays already exported stay;
        nothing is exported on the way out)."""
        if self._finalizer is not None:
            self._finalizer()
            self._finalizer = None
            self._handle = None

    # -- host views ---------------------------------------------------------------
    def _export_all(self):
        if all(self._host.get(k) is not None for k in _ARRAYS):
            return
        lib = _lib.load()
        slots, n_pad = self.stored_slots, self.n_rows_padded
        arr = {
            "cs": np.empty(self.n_chunks + 1, OFFSET_DTYPE),
            "cl": np.empty(self.n_chunks, INDEX_DTYPE),
            "col": np.empty(slots, INDEX_DTYPE),
            "val": np.empty(slots, self.dtype),
            "perm": np.empty(self.n_rows, INDEX_DTYPE),
            "row_lengths": np.empty(n_pad, INDEX_DTYPE),
        }
        _lib.check(lib.sellb_export(
            self._handle, _lib.ptr(arr["cs"]), _lib.ptr(arr["cl"]),
            _lib.ptr(arr["col"]), _lib.ptr(arr["val"]), _lib.ptr(arr["perm"]),
            _lib.ptr(arr["row_lengths"]), None, 0))
        for k, v in arr.items():
            v.flags.writeable = False
            self._host[k] = v

    def _get(self, name):
        a = self._host.get(name)
        if a is None:
            self._export_all()
            a = self._host[name]
        return a

    cs = property(lambda self: self._get("cs"))
    cl = property(lambda self: self._get("cl"))
    col = property(lambda self: self._get("col"))
    val = property(lambda self: self._get("val"))
    perm = property(lambda self: self._get("perm"))
    row_lengths = property(lambda self: self._get("row_lengths"))

    @property
    def nnz(self):
        if self._nnz is None or self._nnz < 0:
            self._nnz = int(self.row_lengths.sum(dtype=np.int64))
        return self._nnz

    @property
    def shape(self):
        return (self.n_rows, self.n_cols)

    @property
    def stored_slots(self):
        if self._slots is None:
            cs = self._host["cs"]
            self._slots = int(cs[-1]) if len(cs) else 0
        return self._slots

    @property
    def inv_perm(self):
        """Stored -> original row (formats.py:265-271)."""
        if self._inv_perm is None:
            inv = np.empty(self.n_rows, dtype=INDEX_DTYPE)
            inv[self.perm] = np.arange(self.n_rows, dtype=INDEX_DTYPE)
            self._inv_perm = inv
        return self._inv_perm

    def __repr__(self):
        return (f"SellMatrix(n_rows={self.n_rows}, n_cols={self.n_cols}, C={self.C}, "
                f"sigma={self.sigma}, n_chunks={self.n_chunks}, "
                f"slots={self.stored_slots}, device={self.device})")


def _free_handle(handle):
    try:
        _lib.load().sellb_free(handle)
    except Exception:   # interpreter shutdown
        pass


def chunk_occupancy(m):
    """beta = nnz / stored slots; 1.0 when nothing is stored
    (formats.py:274-282)."""
    slots = m.stored_slots
    return 1.0 if slots == 0 else m.nnz / slots


def crs_to_sell(m, C, sigma, align_bytes=1, permute_cols=False, *, device=0,
                dtype=None, stream=None):
    """Build SELL-C-sigma from CRS on the GPU (formats.py:295-393).

    Rows are sorted by non-increasing length within sigma-scopes (stable on
    the original index), padded to a multiple of C, each chunk padded to its
    longest row (optionally rounded so C*cl*4 is a multiple of 64 bytes), and
    columns optionally permuted into stored-row space.  Arrays and the
    permutation are bit-identical to the reference's.

    Extensions (keyword-only): ``device`` (CUDA ordinal), ``dtype``
    (np.float32 builds an fp32 matrix from the fp64 values, rounding once),
    ``stream`` (a cudaStream_t as int; None = default stream).
    """
    # the reference's checks, in its order (formats.py:309-319)
    if C < 1:
        raise ParameterError(f"chunk height C must be >= 1, got {C}")
    if sigma < 1:
        raise ParameterError(f"sigma must be >= 1, got {sigma}")
    if align_bytes not in (1, 64):
        raise ParameterError(f"align_bytes must be 1 or 64, got {align_bytes}")
    if permute_cols and m.n_rows != m.n_cols:
        raise ParameterError(
            "column permutation requires a square matrix "
            f"(got {m.n_rows}x{m.n_cols}); rows and columns share one index space")
    n = m.n_rows
    if C < sigma < n and sigma % C:
        raise ParameterError(
            f"sigma ({sigma}) must be a multiple of C ({C}) when C < sigma < n_rows")
    lib = _lib.require_device()
    val = m.val
    if dtype is not None and np.dtype(dtype) == np.float32:
        val = np.ascontiguousarray(val, dtype=np.float32)
    dt = _lib.SELLB_F32 if val.dtype == np.float32 else _lib.SELLB_F64
    out = ctypes.c_void_p()
    _lib.check(lib.sellb_build_from_crs(
        _lib.ptr(m.rpt), _lib.ptr(m.col), _lib.ptr(val), dt, m.n_rows, m.n_cols,
        int(C), int(sigma), int(align_bytes), int(bool(permute_cols)), int(device),
        stream, 0, ctypes.byref(out)))
    return SellMatrix._adopt(out.value, sigma)


def crs_to_sell_device(rpt, col, val, n_rows, n_cols, C, sigma, align_bytes=1,
                       permute_cols=False, *, device=0, stream=None):
    """Device-input build: rpt/col/val are CUDA tensors (torch) or raw device
    pointers already on ``device`` -- no host round trip (used by the
    multi-GPU path and the benchmark's large configs)."""
    if C < 1 or sigma < 1 or align_bytes not in (1, 64):
        raise ParameterError("invalid C / sigma / align_bytes")
    if C < sigma < n_rows and sigma % C:
        raise ParameterError(
            f"sigma ({sigma}) must be a multiple of C ({C}) when C < sigma < n_rows")
    lib = _lib.require_device()
    is_f32 = (getattr(val, "dtype", None) is not None and "float32" in str(val.dtype))
    dt = _lib.SELLB_F32 if is_f32 else _lib.SELLB_F64
    out = ctypes.c_void_p()
    _lib.check(lib.sellb_build_from_crs(
        _lib.ptr(rpt) if not isinstance(rpt, int) else rpt,
        _lib.ptr(col) if not isinstance(col, int) else col,
        _lib.ptr(val) if not isinstance(val, int) else val,
        dt, int(n_rows), int(n_cols), int(C), int(sigma), int(align_bytes),
        int(bool(permute_cols)), int(device), stream, 1, ctypes.byref(out)))
    return SellMatrix._adopt(out.value, sigma)


def sell_to_ellpack(m, **kw):
    """ELLPACK = SELL-N-1, a single chunk (formats.py:396-399)."""
    return crs_to_sell(m, C=max(m.n_rows, 1), sigma=1, **kw)


def sell_to_crs(m):
    """Inverse conversion: strip padding, undo the row (and column)
    permutation (formats.py:402-420).  Host-side format utility."""
    lens = m.row_lengths[m.perm].astype(OFFSET_DTYPE) if m.n_rows else \
        np.zeros(0, OFFSET_DTYPE)
    rpt = np.zeros(m.n_rows + 1, OFFSET_DTYPE)
    np.cumsum(lens, out=rpt[1:])
    nnz = int(rpt[-1])
    if nnz:
        stored = np.repeat(m.perm.astype(OFFSET_DTYPE), lens)
        j = np.arange(nnz, dtype=OFFSET_DTYPE) - np.repeat(rpt[:-1], lens)
        flat = m.cs[stored // m.C] + j * m.C + stored % m.C
        cols = m.col[flat].astype(OFFSET_DTYPE)
        if m.col_permuted:
            cols = m.inv_perm[cols].astype(OFFSET_DTYPE)
        vals = m.val[flat]
    else:
        cols = np.zeros(0, OFFSET_DTYPE)
        vals = np.zeros(0, VALUE_DTYPE)
    rows = np.repeat(np.arange(m.n_rows, dtype=OFFSET_DTYPE), lens)
    return coo_to_crs(COOMatrix(m.n_rows, m.n_cols, rows, cols, vals))


def permute_vector(v, perm):
    """original -> stored order: out[perm[i]] = v[i] (formats.py:423-430)."""
    v = np.asarray(v, dtype=VALUE_DTYPE)
    if len(v) != len(perm):
        raise DimensionError(f"vector length {len(v)} != permutation length {len(perm)}")
    out = np.empty_like(v)
    out[perm] = v
    return out


def unpermute_vector(v, perm):
    """stored -> original order: out[i] = v[perm[i]]; padding dropped
    (formats.py:433-441)."""
    v = np.asarray(v, dtype=VALUE_DTYPE)
    if len(v) < len(perm):
        raise DimensionError(f"vector length {len(v)} < permutation length {len(perm)}")
    return v[perm]
