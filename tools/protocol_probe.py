"""The reference kernels protocol (kernels_cuda.spmv_sell_range on host
arrays, _kernels.pyx:65-92): a handle imported without row_lengths (pad-
inclusive only) vs the same handle after sellb_infer_row_lengths (what
kernels_cuda now does on import): device-only SpMV time and the host-array
call's time.  python tools/protocol_probe.py [cfg] [sigma]"""
import ctypes
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import oracle  # noqa: E402
from bench import make_matrix  # noqa: E402
from paper_1307_6209_b200 import _lib, generate  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg3"
sigma = int(sys.argv[2]) if len(sys.argv) > 2 else 1
m, desc = make_matrix(cfg)
o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, 32, sigma)
lib = _lib.load()
x = generate.rhs(m.n_cols)
y_ref = oracle.spmv_sell(o, x, threads=os.cpu_count() or 1)
xd = torch.from_numpy(x).cuda()
nnz = int(m.rpt[-1])
for infer in (False, True):
    h = ctypes.c_void_p()
    _lib.check(lib.sellb_import(_lib.ptr(o.cs), _lib.ptr(o.cl), _lib.ptr(o.col), _lib.ptr(o.val),
                                None, None, _lib.SELLB_F64, o.n_chunks * 32, m.n_cols, 32, 1,
                                o.n_chunks, len(o.val), 0, 0, None, 0, ctypes.byref(h)))
    t0 = time.perf_counter()
    if infer:
        _lib.check(lib.sellb_infer_row_lengths(h, None))
    t_inf = time.perf_counter() - t0
    yd = torch.zeros(o.n_chunks * 32, dtype=torch.float64, device="cuda")
    for _ in range(5):
        _lib.check(lib.sellb_spmv(h, xd.data_ptr(), yd.data_ptr(), 0, o.n_chunks, 0, 0, None))
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        _lib.check(lib.sellb_spmv(h, xd.data_ptr(), yd.data_ptr(), 0, o.n_chunks, 0, 0, None))
    e1.record()
    e1.synchronize()
    dev_ms = e0.elapsed_time(e1) / 50
    ok_dev = yd.cpu().numpy().tobytes() == y_ref.tobytes()
    y = np.zeros(o.n_chunks * 32)
    for _ in range(3):
        _lib.check(lib.sellb_spmv_host(h, _lib.ptr(x), _lib.ptr(y), 0, o.n_chunks, 0, 0, None))
    t0 = time.perf_counter()
    for _ in range(20):
        _lib.check(lib.sellb_spmv_host(h, _lib.ptr(x), _lib.ptr(y), 0, o.n_chunks, 0, 0, None))
    host_ms = (time.perf_counter() - t0) / 20 * 1e3
    ok_host = y.tobytes() == y_ref.tobytes()
    print(f"{desc} sigma={sigma} infer={infer}: infer {t_inf*1e3:.1f} ms; device SpMV "
          f"{dev_ms:.4f} ms = {2*nnz/dev_ms/1e6:.1f} GF/s (bitwise {ok_dev}); host-array call "
          f"{host_ms:.3f} ms = {2*nnz/host_ms/1e6:.1f} GF/s (bitwise {ok_host})", flush=True)
    lib.sellb_free(h)
