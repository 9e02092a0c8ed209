"""ctypes binding of libsellb200.so (the C ABI declared in include/sellb.h).

The library is built in-tree (``paper_1307_6209_b200/libsellb200.so``, see
csrc/Makefile).  There is no CPU fallback: if the library or a CUDA device is
missing, every compute entry point raises ``ResourceError``.
"""

import ctypes
import os
import threading

from .errors import (DimensionError, FormatError, ParameterError, ResourceError,
                     StructuralError)

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("SELLB_LIB_PATH") or os.path.join(HERE, "libsellb200.so")

SELLB_F64 = 0
SELLB_F32 = 1
VARIANT_AUTO = 0
VARIANT_PAD_SKIP = 1
VARIANT_PAD_INCL = 2
ORDER_STORED = 0
ORDER_ORIGINAL = 1

# every symbol include/sellb.h declares (checked by tests/test_abi.py)
EXPORTED = (
    "sellb_last_error", "sellb_version", "sellb_device_count",
    "sellb_build_from_crs", "sellb_import", "sellb_info", "sellb_device_arrays",
    "sellb_export", "sellb_set_variant", "sellb_free", "sellb_spmv",
    "sellb_spmv_chunk_list", "sellb_spmv_host", "sellb_spmv_sell_range_host",
    "sellb_spmv_crs_range_host", "sellb_spmv_crs", "sellb_chunk_occupancy",
    "sellb_sector_occupancy", "sellb_read_sum", "sellb_copy", "sellb_l2_flush",
    "sellb_host_alloc", "sellb_host_free", "sellb_gather", "sellb_scatter",
    "sellb_pad_fixup", "sellb_gen_hamiltonian_rpt", "sellb_gen_hamiltonian_fill",
    "sellb_export_range", "sellb_infer_row_lengths", "sellb_chunk_flags",
    "sellb_coo_to_crs", "sellb_mm_parse_body", "sellb_mm_format_body",
    "sellb_launch_count", "sellb_long_info", "sellb_streamed_bytes",
    "sellb_lru_stream_misses", "sellb_sell_x_lines", "sellb_host_register",
    "sellb_host_unregister", "sellb_set_packed", "sellb_set_shadow", "sellb_crs_import", "sellb_crs_spmv_host",
    "sellb_crs_free", "sellb_gen_powerlaw_rpt", "sellb_gen_powerlaw_fill",
)


class Info(ctypes.Structure):
    _fields_ = [
        ("n_rows", ctypes.c_int64), ("n_cols", ctypes.c_int64),
        ("C", ctypes.c_int64), ("sigma", ctypes.c_int64),
        ("sigma_eff", ctypes.c_int64), ("n_rows_padded", ctypes.c_int64),
        ("n_chunks", ctypes.c_int64), ("slots", ctypes.c_int64),
        ("nnz", ctypes.c_int64), ("dtype", ctypes.c_int32),
        ("device", ctypes.c_int32), ("col_permuted", ctypes.c_int32),
        ("variant", ctypes.c_int32), ("has_row_lengths", ctypes.c_int32),
        ("max_cl", ctypes.c_int32), ("packed", ctypes.c_int32),
        ("shadow", ctypes.c_int32),
    ]


class DevArrays(ctypes.Structure):
    _fields_ = [(name, ctypes.c_void_p) for name in
                ("cs", "cl", "col", "val", "perm", "order", "row_lengths")]


_vp = ctypes.c_void_p
_i64 = ctypes.c_int64
_i32 = ctypes.c_int32

_PROTOS = {
    "sellb_last_error": (ctypes.c_char_p, []),
    "sellb_version": (ctypes.c_int, []),
    "sellb_device_count": (ctypes.c_int, [ctypes.POINTER(_i32)]),
    "sellb_build_from_crs": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i64, _i64, _i32, _i64,
                                            _i32, _i32, _i32, _vp, _i32, ctypes.POINTER(_vp)]),
    "sellb_import": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _i32, _i64, _i64, _i32,
                                    _i64, _i64, _i64, _i32, _i32, _vp, _i32,
                                    ctypes.POINTER(_vp)]),
    "sellb_info": (ctypes.c_int, [_vp, ctypes.POINTER(Info)]),
    "sellb_device_arrays": (ctypes.c_int, [_vp, ctypes.POINTER(DevArrays)]),
    "sellb_export": (ctypes.c_int, [_vp, _vp, _vp, _vp, _vp, _vp, _vp, _vp, _i32]),
    "sellb_set_variant": (ctypes.c_int, [_vp, _i32]),
    "sellb_set_packed": (ctypes.c_int, [_vp, _i32]),
    "sellb_set_shadow": (ctypes.c_int, [_vp, _i32]),
    "sellb_crs_import": (ctypes.c_int, [_vp, _vp, _vp, _i32, _i64, _i64, _i64, _i32,
                                        ctypes.POINTER(_vp)]),
    "sellb_crs_spmv_host": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _i32]),
    "sellb_crs_free": (None, [_vp]),
    "sellb_free": (None, [_vp]),
    "sellb_spmv": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp]),
    "sellb_spmv_chunk_list": (ctypes.c_int, [_vp, _vp, _i64, _vp, _vp, _i32, _vp]),
    "sellb_spmv_host": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i32, _i32, _vp]),
    "sellb_spmv_sell_range_host": (ctypes.c_int, [_vp, _vp, _i32, _vp, _vp, _i64, _i64, _vp,
                                                  _i64, _vp, _i64, _i64, _i64, _i32, _i32]),
    "sellb_spmv_crs_range_host": (ctypes.c_int, [_vp, _i64, _vp, _vp, _i64, _vp, _i64, _vp,
                                                 _i64, _i64, _i32, _i32, _i32]),
    "sellb_spmv_crs": (ctypes.c_int, [_vp, _vp, _vp, _i32, _vp, _vp, _i64, _i64, _i32, _i32,
                                      _vp]),
    "sellb_chunk_occupancy": (ctypes.c_double, [_vp]),
    "sellb_sector_occupancy": (ctypes.c_int, [_vp, ctypes.POINTER(ctypes.c_double),
                                              ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                              _vp]),
    "sellb_read_sum": (ctypes.c_int, [_vp, _i64, ctypes.POINTER(ctypes.c_double), _vp]),
    "sellb_copy": (ctypes.c_int, [_vp, _vp, _i64, _vp]),
    "sellb_l2_flush": (ctypes.c_int, [_vp, _i64, _vp]),
    "sellb_host_alloc": (ctypes.c_int, [ctypes.c_size_t, ctypes.POINTER(_vp)]),
    "sellb_gather": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "sellb_scatter": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i32, _vp]),
    "sellb_pad_fixup": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "sellb_gen_hamiltonian_rpt": (ctypes.c_int, [_i64, _i64, _i64, _vp, _i32, ctypes.c_double,
                                                 ctypes.c_uint64, _vp, ctypes.POINTER(_i64),
                                                 _vp]),
    "sellb_gen_hamiltonian_fill": (ctypes.c_int, [_i64, _i64, _i64, _vp, _i32, ctypes.c_double,
                                                  ctypes.c_uint64, _vp, _vp, _vp, _i32, _vp]),
    "sellb_host_free": (ctypes.c_int, [_vp]),
    "sellb_gen_powerlaw_rpt": (ctypes.c_int, [_i64, _i64, _i64, ctypes.c_double, _i64,
                                              ctypes.c_uint64, _vp, ctypes.POINTER(_i64), _vp]),
    "sellb_gen_powerlaw_fill": (ctypes.c_int, [_i64, _i64, _i64, ctypes.c_double, _i64, _i64,
                                               ctypes.c_uint64, _vp, _vp, _vp, _i32, _vp]),
    "sellb_host_register": (ctypes.c_int, [_vp, ctypes.c_size_t]),
    "sellb_host_unregister": (ctypes.c_int, [_vp]),
    "sellb_export_range": (ctypes.c_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "sellb_infer_row_lengths": (ctypes.c_int, [_vp, _vp]),
    "sellb_chunk_flags": (ctypes.c_int, [_vp, _vp, _vp, _vp]),
    "sellb_coo_to_crs": (ctypes.c_int, [_vp, _vp, _vp, _i64, _i64, _i64, _vp, _vp, _vp,
                                        ctypes.POINTER(_i64), _i32, _vp, _i32]),
    "sellb_launch_count": (_i64, []),
    "sellb_lru_stream_misses": (ctypes.c_int, [_vp, _i64, _i64, _i64, _i32, _vp, _vp]),
    "sellb_sell_x_lines": (ctypes.c_int, [_vp, _i32, _vp, ctypes.POINTER(_i64), _vp]),
    "sellb_streamed_bytes": (ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                            ctypes.POINTER(_i64), _vp]),
    "sellb_long_info": (ctypes.c_int, [_vp, ctypes.POINTER(_i64), ctypes.POINTER(_i64),
                                       ctypes.POINTER(_i64), ctypes.POINTER(_i64)]),
    "sellb_mm_parse_body": (ctypes.c_int, [_vp, _i64, _i32, _i64, _vp, ctypes.POINTER(_i64),
                                           _i32]),
    "sellb_mm_format_body": (ctypes.c_int, [_vp, _vp, _vp, _i64, _vp, _i64,
                                            ctypes.POINTER(_i64), _i32]),
}

_lib = None
_lock = threading.Lock()
_device_count = None


def load():
    """Load the library (no device needed).  Raises ResourceError if the
    shared object is missing or does not load."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise ResourceError(
                    f"CUDA library {LIB_PATH} is not built; run "
                    "`python -c 'import __graft_entry__ as g; g.build()'` or "
                    "`make -C paper_1307_6209_b200/csrc`")
            try:
                lib = ctypes.CDLL(LIB_PATH)
            except OSError as exc:
                raise ResourceError(f"cannot load {LIB_PATH}: {exc}") from exc
            for name, (res, args) in _PROTOS.items():
                if not hasattr(lib, name):      # older builds under SELLB_LIB_PATH
                    continue
                fn = getattr(lib, name)
                fn.restype = res
                fn.argtypes = args
            _lib = lib
    return _lib


def device_count():
    global _device_count
    if _device_count is None:
        n = _i32(0)
        rc = load().sellb_device_count(ctypes.byref(n))
        _device_count = int(n.value) if rc == 0 else 0
    return _device_count


def require_device():
    """The product path: fail loudly without a GPU (no CPU fallback)."""
    if device_count() < 1:
        raise ResourceError("no CUDA device is visible; the sell-b200 backend "
                            "has no CPU fallback")
    return load()


def last_error():
    msg = load().sellb_last_error()
    return msg.decode(errors="replace") if msg else ""


_ERRORS = {-1: ParameterError, -2: DimensionError, -3: StructuralError,
           -4: ResourceError, -5: FormatError}


def check(rc):
    if rc == 0:
        return
    exc = _ERRORS.get(rc, ResourceError)
    raise exc(last_error() or f"sellb error {rc}")


def ptr(a):
    """Address of a NumPy array or torch tensor (None -> NULL)."""
    if a is None:
        return None
    if hasattr(a, "data_ptr"):
        return a.data_ptr()
    return a.ctypes.data
