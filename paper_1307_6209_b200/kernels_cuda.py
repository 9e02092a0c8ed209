"""The ``cuda`` kernels module: the reference's backend protocol on the GPU.

The reference selects a kernels module (backend.py:32-47) and calls seven
attributes on it from spmv.py, bench.py, membench.py and cachesim.py.  This
module implements them with libsellb200.so so it can be passed as
``kernels=`` to the reference's own API (``sellkit.spmv_sell(m, x,
kernels=paper_1307_6209_b200.get_kernels("cuda"))``) or registered in the
reference's test fixture (tests/conftest.py:38-43).

    NAME                      "cuda"
    spmv_sell_range           _kernels.pyx:65-92   (pad-inclusive, bitwise equal)
    spmv_crs_range            _kernels.pyx:17-31   (bitwise equal)
    spmv_crs_unrolled_range   _kernels.pyx:34-62   (bitwise equal)
    read_sum                  _kernels.pyx:142-161 (device reduction; rounding differs)
    copy_array                _kernels.pyx:164-170
    lru_stream_misses         _kernels.pyx:95-139  (LRU stack distances on the
                              device, equal miss counts)

Arrays are host NumPy buffers, as in the reference.  Matrix arrays (SELL
and CRS alike) are uploaded once and cached by buffer identity (containers
are immutable, formats.py:7); the cache entry dies with the ``val`` array.  Every call
blocks until y is back on the host, like the reference's nogil loops.
"""

import threading
import weakref

import numpy as np

from . import _lib
from .errors import ParameterError, ResourceError

NAME = "cuda"

_cache = {}
_cache_lock = threading.Lock()


def _free(handle):
    try:
        _lib.load().sellb_free(handle)
    except Exception:
        pass


def _evict(key):
    with _cache_lock:
        h = _cache.pop(key, None)
    if h is not None:
        _free(h)


def _sell_handle(cs, cl, C, col, val, n_cols):
    key = (cs.ctypes.data, len(cs), cl.ctypes.data, col.ctypes.data,
           val.ctypes.data, len(val), int(C), int(n_cols))
    with _cache_lock:
        h = _cache.get(key)
    if h is not None:
        return h
    import ctypes
    lib = _lib.require_device()
    n_chunks = len(cl)
    out = ctypes.c_void_p()
    _lib.check(lib.sellb_import(
        _lib.ptr(cs), _lib.ptr(cl), _lib.ptr(col), _lib.ptr(val), None, None,
        _lib.SELLB_F64, n_chunks * int(C), int(n_cols), int(C), 1, n_chunks, len(val), 0,
        0, None, 0, ctypes.byref(out)))
    h = out.value
    # the protocol passes no row_lengths: infer them from each row's trailing
    # (0.0, column 0) slots -- the .sell reader's rule (io.py) -- so the
    # pad-skipping kernels, long-row roles and shadow layout apply.  Bitwise
    # the same y: a real trailing (0.0, col 0) entry adds 0*x[0], which the
    # pad term adds once instead (a no-op for finite x[0], NaN otherwise).
    try:
        _lib.check(lib.sellb_infer_row_lengths(h, None))
    except Exception:
        _free(h)
        raise
    try:
        weakref.finalize(val.base if val.base is not None else val, _evict, key)
    except TypeError:
        pass
    with _cache_lock:
        if key in _cache:          # another thread won the race
            _free(h)
            return _cache[key]
        _cache[key] = h
    return h


def _c64(a, dtype):
    a = np.asarray(a)
    if a.dtype != dtype or not a.flags.c_contiguous:
        raise ParameterError(f"expected a contiguous {np.dtype(dtype).name} buffer")
    return a


def spmv_sell_range(cs, cl, C, col, val, x, y, c0, c1, accumulate):
    """y[c0*C:c1*C] (+)= chunk rows of A @ x (_kernels.pyx:65-92)."""
    if c1 <= c0:
        return
    cs, cl = _c64(cs, np.int64), _c64(cl, np.int32)
    col, val = _c64(col, np.int32), _c64(val, np.float64)
    x, y = _c64(x, np.float64), _c64(y, np.float64)
    if not y.flags.writeable:
        raise ParameterError("y must be writable")
    if c0 < 0 or c1 > len(cl) or len(y) < len(cl) * int(C):
        raise ParameterError("chunk range or y length out of bounds")
    h = _sell_handle(cs, cl, C, col, val, len(x))
    _lib.check(_lib.load().sellb_spmv_host(h, _lib.ptr(x), _lib.ptr(y), int(c0),
                                           int(c1), int(bool(accumulate)),
                                           _lib.ORDER_STORED, None))


def _crs_handle(rpt, col, val, n_cols):
    key = ("crs", rpt.ctypes.data, len(rpt), col.ctypes.data, val.ctypes.data, len(val),
           int(n_cols))
    with _cache_lock:
        h = _cache.get(key)
    if h is not None:
        return h
    import ctypes
    lib = _lib.require_device()
    out = ctypes.c_void_p()
    _lib.check(lib.sellb_crs_import(_lib.ptr(rpt), _lib.ptr(col), _lib.ptr(val),
                                    _lib.SELLB_F64, len(rpt) - 1, int(n_cols), len(val), 0,
                                    ctypes.byref(out)))
    h = out.value
    try:
        weakref.finalize(val.base if val.base is not None else val, _evict_crs, key)
    except TypeError:
        pass
    with _cache_lock:
        if key in _cache:
            _lib.load().sellb_crs_free(h)
            return _cache[key]
        _cache[key] = h
    return h


def _evict_crs(key):
    with _cache_lock:
        h = _cache.pop(key, None)
    if h is not None:
        try:
            _lib.load().sellb_crs_free(h)
        except Exception:
            pass


def _crs(rpt, col, val, x, y, r0, r1, accumulate, unrolled):
    if r1 <= r0:
        return
    rpt, col = _c64(rpt, np.int64), _c64(col, np.int32)
    val, x, y = _c64(val, np.float64), _c64(x, np.float64), _c64(y, np.float64)
    if not y.flags.writeable:
        raise ParameterError("y must be writable")
    if r0 < 0 or r1 > len(rpt) - 1 or len(y) < len(rpt) - 1:
        raise ParameterError("row range or y length out of bounds")
    h = _crs_handle(rpt, col, val, len(x))
    _lib.check(_lib.load().sellb_crs_spmv_host(h, _lib.ptr(x), _lib.ptr(y), int(r0), int(r1),
                                               int(bool(accumulate)), int(unrolled)))


def spmv_crs_range(rpt, col, val, x, y, r0, r1, accumulate):
    """_kernels.pyx:17-31, one thread per row, reference summation order."""
    _crs(rpt, col, val, x, y, r0, r1, accumulate, False)


def spmv_crs_unrolled_range(rpt, col, val, x, y, r0, r1, accumulate):
    """_kernels.pyx:34-62, four partial sums combined ((t0+t1)+t2)+t3."""
    _crs(rpt, col, val, x, y, r0, r1, accumulate, True)


def read_sum(a):
    """Sum of a float64 buffer on the device (membench read kernel)."""
    import ctypes
    import torch
    lib = _lib.require_device()
    t = torch.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).cuda()
    out = ctypes.c_double(0.0)
    _lib.check(lib.sellb_read_sum(t.data_ptr(), t.numel(), ctypes.byref(out),
                                  torch.cuda.current_stream().cuda_stream))
    return float(out.value)


def copy_array(src, dst):
    """dst[:] = src through the device copy kernel."""
    import torch
    src = np.ascontiguousarray(src, dtype=np.float64)
    if len(dst) != len(src):
        raise ValueError("source and destination lengths differ")
    lib = _lib.require_device()
    s = torch.from_numpy(src).cuda()
    d = torch.empty_like(s)
    _lib.check(lib.sellb_copy(s.data_ptr(), d.data_ptr(), s.numel(),
                              torch.cuda.current_stream().cuda_stream))
    dst[:] = d.cpu().numpy()


def lru_stream_misses(lines, cache_lines, n_line_slots):
    """_kernels.pyx:95-139: misses of a fully-associative LRU cache of
    ``cache_lines`` lines replaying the line-id stream, counted on the GPU
    from LRU stack distances (csrc/sellb_lru.cu).  Same result as the
    reference's MRU-list walk; 0 for an empty stream, len(lines) for
    cache_lines <= 0; an id outside [0, n_line_slots) is a ParameterError
    (the reference indexes its table unchecked)."""
    import ctypes
    import torch
    lib = _lib.require_device()
    lines = np.ascontiguousarray(lines, dtype=np.int64)
    out = ctypes.c_int64(0)
    _lib.check(lib.sellb_lru_stream_misses(
        lines.ctypes.data if len(lines) else None, len(lines), int(cache_lines),
        int(n_line_slots), 0, ctypes.byref(out),
        torch.cuda.current_stream().cuda_stream))
    return int(out.value)


def sell_rhs_misses(m, line_bytes, cache_lines, n_line_slots):
    """LRU misses of a device-resident SellMatrix's x stream without a host
    pass: the line ids are extracted on the device (sellb_sell_x_lines) and
    replayed there (sellb_lru_stream_misses)."""
    import ctypes
    import torch
    lib = _lib.require_device()
    st = torch.cuda.current_stream(m.device).cuda_stream
    with torch.cuda.device(m.device):
        lines = torch.empty(max(m.nnz, 1), dtype=torch.int64, device=f"cuda:{m.device}")
        n = ctypes.c_int64(0)
        _lib.check(lib.sellb_sell_x_lines(m.handle, line_bytes // 8, lines.data_ptr(),
                                          ctypes.byref(n), st))
        out = ctypes.c_int64(0)
        _lib.check(lib.sellb_lru_stream_misses(lines.data_ptr(), n.value, int(cache_lines),
                                               int(n_line_slots), 1, ctypes.byref(out), st))
    return int(out.value)
