"""TEST INFRASTRUCTURE ONLY -- the CPU checker for the CUDA product path.

NumPy-facing wrapper around ``oracle/liboracle_sell.so`` (the plain-C
restatement in ``sell_oracle.c``) and loader for ``oracle/_ref`` (the
reference's own Cython kernel core compiled from /root/reference sources by
``build_ref.sh``).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may import this module.  The
product package ``paper_1307_6209_b200`` never imports it: the CUDA path fails
loudly instead of falling back to the CPU.

Each function names the reference code it restates (paths relative to
/root/reference/pkg/src/sellkit).  Parity pin: tests/test_oracle_golden.py
checks this module against vectors the reference produced
(tests/golden/make_golden.py).
"""

import ctypes
import glob
import importlib.util
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle_sell.so")
REF_DIR = os.path.join(HERE, "_ref")

_lib = None

_i64p = ctypes.POINTER(ctypes.c_int64)
_i32p = ctypes.POINTER(ctypes.c_int32)
_f64p = ctypes.POINTER(ctypes.c_double)
_f32p = ctypes.POINTER(ctypes.c_float)
_i64 = ctypes.c_int64


def build():
    """Compile liboracle_sell.so (gcc, no FMA)."""
    import subprocess
    subprocess.check_call(["make", "-s", "-C", HERE, "liboracle_sell.so"])


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH) or (
                os.path.getmtime(LIB_PATH)
                < os.path.getmtime(os.path.join(HERE, "sell_oracle.c"))):
            build()
        L = ctypes.CDLL(LIB_PATH)
        L.oracle_sigma_eff.restype = _i64
        L.oracle_sigma_eff.argtypes = [_i64, _i64, _i64]
        L.oracle_sell_plan.restype = ctypes.c_int
        L.oracle_sell_plan.argtypes = [_i64p, _i64, _i64, _i64, _i64, _i64p,
                                       _i32p, _i32p, _i32p, _i64p]
        L.oracle_sell_fill.restype = ctypes.c_int
        L.oracle_sell_fill.argtypes = [_i64p, _i32p, _f64p, _i64, _i64, _i64p,
                                       _i32p, _i32p, _i64p, ctypes.c_int,
                                       _i32p, _f64p]
        L.oracle_sell_fill_f32.restype = ctypes.c_int
        L.oracle_sell_fill_f32.argtypes = [_i64p, _i32p, _f32p, _i64, _i64,
                                           _i64p, _i32p, _i32p, _i64p,
                                           ctypes.c_int, _i32p, _f32p]
        L.oracle_spmv_sell_range.restype = ctypes.c_int
        L.oracle_spmv_sell_range.argtypes = [_i64p, _i32p, _i64, _i32p, _f64p,
                                             _f64p, _f64p, _i64, _i64,
                                             ctypes.c_int]
        L.oracle_spmv_sell_range_f32.restype = ctypes.c_int
        L.oracle_spmv_sell_range_f32.argtypes = [_i64p, _i32p, _i64, _i32p,
                                                 _f32p, _f32p, _f32p, _i64,
                                                 _i64, ctypes.c_int]
        for name in ("oracle_spmv_crs_range", "oracle_spmv_crs_unrolled_range"):
            f = getattr(L, name)
            f.restype = ctypes.c_int
            f.argtypes = [_i64p, _i32p, _f64p, _f64p, _f64p, _i64, _i64,
                          ctypes.c_int]
        L.oracle_read_sum.restype = ctypes.c_double
        L.oracle_read_sum.argtypes = [_f64p, _i64]
        L.oracle_coo_to_crs.restype = _i64
        L.oracle_coo_to_crs.argtypes = [_i64p, _i64p, _f64p, _i64, _i64, _i64p, _i32p,
                                        _f64p]
        L.oracle_lru_stream_misses.restype = _i64
        L.oracle_lru_stream_misses.argtypes = [_i64p, _i64, _i64, _i64]
        _lib = L
    return _lib


def _p(a, t):
    return a.ctypes.data_as(t)


class OracleSell:
    """Plain record of the SELL-C-sigma arrays (SellMatrix fields,
    formats.py:183-207)."""

    def __init__(self, **kw):
        self.__dict__.update(kw)

    @property
    def nnz(self):
        return int(self.row_lengths.sum(dtype=np.int64))

    @property
    def stored_slots(self):
        return int(self.cs[-1])


def coo_to_crs(rows, cols, vals, n_rows):
    """canonicalize_coo + coo_to_crs (formats.py:89-108,169-175): returns
    (rpt int64, col int32, val f64).  Indices must be in bounds."""
    rows = np.ascontiguousarray(rows, np.int64)
    cols = np.ascontiguousarray(cols, np.int64)
    vals = np.ascontiguousarray(vals, np.float64)
    nnz = len(vals)
    rpt = np.zeros(n_rows + 1, np.int64)
    col = np.zeros(max(nnz, 1), np.int32)
    val = np.zeros(max(nnz, 1))
    u = lib().oracle_coo_to_crs(_p(rows, _i64p), _p(cols, _i64p), _p(vals, _f64p), nnz,
                                n_rows, _p(rpt, _i64p), _p(col, _i32p), _p(val, _f64p))
    if u < 0:
        raise MemoryError("oracle_coo_to_crs")
    return rpt, col[:u].copy(), val[:u].copy()


def sigma_eff(n_rows, C, sigma):
    """formats.py:321-334 (returns -1 for the ParameterError case)."""
    return int(lib().oracle_sigma_eff(n_rows, C, sigma))


def crs_to_sell(rpt, col, val, n_rows, n_cols, C, sigma, align_bytes=1,
                permute_cols=False):
    """formats.py:295-393 restated in C.  Raises ValueError where the
    reference raises ParameterError."""
    if permute_cols and n_rows != n_cols:
        raise ValueError("column permutation requires a square matrix")
    rpt = np.ascontiguousarray(rpt, dtype=np.int64)
    col = np.ascontiguousarray(col, dtype=np.int32)
    f32 = np.asarray(val).dtype == np.float32
    val = np.ascontiguousarray(val, dtype=np.float32 if f32 else np.float64)
    n = int(n_rows)
    n_pad = ((n + C - 1) // C) * C if n and C >= 1 else 0
    n_chunks = n_pad // C if C >= 1 else 0
    order = np.empty(max(n_pad, 1), np.int64)
    perm = np.empty(max(n, 1), np.int32)
    row_lengths = np.empty(max(n_pad, 1), np.int32)
    cl = np.empty(max(n_chunks, 1), np.int32)
    cs = np.empty(n_chunks + 1, np.int64)
    L = lib()
    st = L.oracle_sell_plan(_p(rpt, _i64p), n, C, sigma, align_bytes,
                            _p(order, _i64p), _p(perm, _i32p),
                            _p(row_lengths, _i32p), _p(cl, _i32p),
                            _p(cs, _i64p))
    if st != 0:
        raise ValueError(f"invalid SELL parameters (C={C}, sigma={sigma}, "
                         f"align_bytes={align_bytes})")
    total = int(cs[n_chunks])
    out_col = np.empty(max(total, 1), np.int32)
    out_val = np.empty(max(total, 1), val.dtype)
    fill = L.oracle_sell_fill_f32 if f32 else L.oracle_sell_fill
    vp = _f32p if f32 else _f64p
    fill(_p(rpt, _i64p), _p(col, _i32p), _p(val, vp), n, C, _p(order, _i64p),
         _p(perm, _i32p), _p(row_lengths, _i32p), _p(cs, _i64p),
         int(bool(permute_cols)), _p(out_col, _i32p), _p(out_val, vp))
    return OracleSell(
        n_rows=n, n_cols=int(n_cols), C=int(C), sigma=int(sigma),
        n_rows_padded=n_pad, n_chunks=n_chunks, cs=cs, cl=cl[:n_chunks],
        col=out_col[:total], val=out_val[:total], perm=perm[:n],
        row_lengths=row_lengths[:n_pad], order=order[:n_pad],
        col_permuted=bool(permute_cols))


def spmv_sell_range(cs, cl, C, col, val, x, y, c0, c1, accumulate):
    """_kernels.pyx:65-92 (fp64) or its binary32 analogue."""
    L = lib()
    if val.dtype == np.float32:
        st = L.oracle_spmv_sell_range_f32(
            _p(cs, _i64p), _p(cl, _i32p), C, _p(col, _i32p), _p(val, _f32p),
            _p(x, _f32p), _p(y, _f32p), c0, c1, int(bool(accumulate)))
    else:
        st = L.oracle_spmv_sell_range(
            _p(cs, _i64p), _p(cl, _i32p), C, _p(col, _i32p), _p(val, _f64p),
            _p(x, _f64p), _p(y, _f64p), c0, c1, int(bool(accumulate)))
    if st != 0:
        raise MemoryError("oracle accumulator allocation failed")


def spmv_sell(s, x, y=None, accumulate=False, threads=1):
    """spmv.py:105-122 with static contiguous chunk spans (spmv.py:53-58).
    Returns y in stored (padded) order."""
    dt = s.val.dtype
    x = np.ascontiguousarray(x, dtype=dt)
    if y is None:
        y = np.zeros(s.n_rows_padded, dt)
    n_units = s.n_chunks
    if threads <= 1 or n_units <= 1:
        spmv_sell_range(s.cs, s.cl, s.C, s.col, s.val, x, y, 0, n_units,
                        accumulate)
        return y
    bounds = np.linspace(0, n_units, threads + 1).astype(int)
    spans = [(int(bounds[t]), int(bounds[t + 1])) for t in range(threads)]
    spans = [sp for sp in spans if sp[1] > sp[0]]
    with ThreadPoolExecutor(max_workers=len(spans)) as pool:
        list(pool.map(lambda sp: spmv_sell_range(
            s.cs, s.cl, s.C, s.col, s.val, x, y, sp[0], sp[1], accumulate),
            spans))
    return y


def spmv_crs_range(rpt, col, val, x, y, r0, r1, accumulate, unrolled=False):
    """_kernels.pyx:17-31 (or :34-62 when unrolled)."""
    f = (lib().oracle_spmv_crs_unrolled_range if unrolled
         else lib().oracle_spmv_crs_range)
    f(_p(rpt, _i64p), _p(col, _i32p), _p(val, _f64p), _p(x, _f64p),
      _p(y, _f64p), r0, r1, int(bool(accumulate)))


def spmv_crs(rpt, col, val, x, n_rows, y=None, accumulate=False,
             unrolled=False):
    x = np.ascontiguousarray(x, dtype=np.float64)
    if y is None:
        y = np.zeros(n_rows)
    spmv_crs_range(np.ascontiguousarray(rpt, np.int64),
                   np.ascontiguousarray(col, np.int32),
                   np.ascontiguousarray(val, np.float64), x, y, 0, n_rows,
                   accumulate, unrolled)
    return y


def read_sum(a):
    """_kernels.pyx:142-161."""
    a = np.ascontiguousarray(a, dtype=np.float64)
    return float(lib().oracle_read_sum(_p(a, _f64p), len(a)))


def lru_stream_misses(lines, cache_lines, n_line_slots):
    """_kernels.pyx:95-139: misses of a fully-associative LRU cache."""
    lines = np.ascontiguousarray(lines, dtype=np.int64)
    r = lib().oracle_lru_stream_misses(_p(lines, _i64p), len(lines), int(cache_lines),
                                       int(n_line_slots))
    if r < 0:
        raise MemoryError("oracle LRU table")
    return int(r)


def unpermute(v, perm):
    """formats.py:433-441."""
    return np.asarray(v)[perm]


def permute(v, perm):
    """formats.py:423-430."""
    v = np.asarray(v)
    out = np.empty_like(v)
    out[perm] = v
    return out


# ---------------------------------------------------------------------------
# The reference's own compiled core (oracle/_ref, built by build_ref.sh)
# ---------------------------------------------------------------------------

_ref_mod = None


def ref_kernels():
    """Import oracle/_ref/_kernels*.so (the reference's _kernels.pyx compiled
    with its own flags).  Returns None when it was not built."""
    global _ref_mod
    if _ref_mod is None:
        hits = glob.glob(os.path.join(REF_DIR, "_kernels*.so"))
        if not hits:
            return None
        spec = importlib.util.spec_from_file_location("_kernels", hits[0])
        mod = importlib.util.module_from_spec(spec)
        spec.loader.exec_module(mod)
        _ref_mod = mod
    return _ref_mod
