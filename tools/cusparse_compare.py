"""Library comparison: our SELL-C-σ kernel vs cuSPARSE
CSR (ALG1, ALG2) and cuSPARSE Sliced-ELL (SELL_ALG1, slice 32) on the same
matrices, same x, same GPU, all device-resident, timed with CUDA events over
`reps` back-to-back launches (inputs > L2 for cfg2/cfg3/cfg4; cfg1 fits in L2
for every arm alike).

cuSPARSE's Sliced-ELL is SELL-32-1 with padding column -1: it gets our own
σ=1 layout (same slices, same column-major order) with pads re-marked.

usage: python tools/cusparse_compare.py [cfg ...] [--f32] > out.json
Prints one JSON line per (config, dtype).  Test infrastructure: the oracle
is used only to check every arm's y.
"""
import ctypes
import json
import os
import subprocess
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import paper_1307_6209_b200 as sb  # noqa: E402
from paper_1307_6209_b200 import generate  # noqa: E402
from paper_1307_6209_b200 import _lib  # noqa: E402
import oracle  # noqa: E402
from bench import make_matrix  # noqa: E402

LIB = os.path.join(ROOT, "tools", "_build", "libcspbench.so")


def build():
    src = os.path.join(ROOT, "tools", "cusparse_bench.cu")
    if os.path.exists(LIB) and os.path.getmtime(LIB) >= os.path.getmtime(src):
        return
    os.makedirs(os.path.dirname(LIB), exist_ok=True)
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3",
                           "-shared", "-Xcompiler", "-fPIC", src, "-lcusparse", "-o", LIB])


def csp(lib, fmt, f32, n_rows, n_cols, nnz, val_size, ptr, col, val, x, y, reps):
    ms = ctypes.c_float()
    rc = lib.csp_spmv(fmt, int(f32), ctypes.c_int64(n_rows), ctypes.c_int64(n_cols),
                      ctypes.c_int64(nnz), ctypes.c_int64(val_size), 32,
                      ctypes.c_void_p(ptr.data_ptr()), ctypes.c_void_p(col.data_ptr()),
                      ctypes.c_void_p(val.data_ptr()), ctypes.c_void_p(x.data_ptr()),
                      ctypes.c_void_p(y.data_ptr()), 10, reps, ctypes.byref(ms))
    if rc:
        raise RuntimeError(f"cusparse arm {fmt} failed ({rc})")
    return ms.value


def ours(s, x, y, reps):
    lib = _lib.load()
    st = torch.cuda.current_stream()
    for _ in range(10):
        _lib.check(lib.sellb_spmv(s.handle, x.data_ptr(), y.data_ptr(), 0, s.n_chunks, 0, 0,
                                  st.cuda_stream))
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record(st)
    for _ in range(reps):
        lib.sellb_spmv(s.handle, x.data_ptr(), y.data_ptr(), 0, s.n_chunks, 0, 0,
                       st.cuda_stream)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / reps


def rel_err(a, ref):
    scale = max(1.0, float(np.max(np.abs(ref)))) if len(ref) else 1.0
    return float(np.max(np.abs(a - ref))) / scale if len(ref) else 0.0


def run(cfg, f32, reps):
    m, desc = make_matrix(cfg)
    dt = np.float32 if f32 else np.float64
    tdt = torch.float32 if f32 else torch.float64
    n, nc, nnz = m.n_rows, m.n_cols, int(m.rpt[-1])
    xh = generate.rhs(nc).astype(dt)
    x = torch.from_numpy(xh).cuda()
    val_h = m.val.astype(dt)
    # reference y: the oracle on the same (dtype-rounded) inputs, fp64 arithmetic
    yref = oracle.spmv_crs(m.rpt, m.col, val_h.astype(np.float64), xh.astype(np.float64), n)
    out = {"config": cfg, "matrix": desc, "dtype": "f32" if f32 else "f64", "n_rows": n,
           "nnz": nnz, "reps": reps, "arms": {}}
    flops = 2.0 * nnz

    def rec(name, ms, y):
        out["arms"][name] = {"ms": round(ms, 5), "gflops": round(flops / ms / 1e6, 1),
                             "max_rel_err": rel_err(y[:n].astype(np.float64), yref)}

    # ours: SELL-32-σ for σ in {1, N} (auto variant)
    for sigma in (1, n):
        s = sb.crs_to_sell(m, 32, sigma, dtype=dt)
        y = torch.zeros(s.n_rows_padded, dtype=tdt, device="cuda")
        ms = ours(s, x, y, reps)
        yo = sb.spmv_sell(s, x, out_order="original").cpu().numpy()
        rec(f"ours_sell32_s{'N' if sigma == n else sigma}", ms, yo)
        if sigma == 1:
            s1 = s
        else:
            s.free()
    # ours: the reference's CRS kernels (bit-exact order) on the same CRS input
    rpt64 = torch.from_numpy(m.rpt).cuda()
    col32 = torch.from_numpy(m.col.astype(np.int32)).cuda()
    valt = torch.from_numpy(val_h).cuda()
    y = torch.zeros(n, dtype=tdt, device="cuda")
    slib = _lib.load()
    code = _lib.SELLB_F32 if f32 else _lib.SELLB_F64
    for unrolled, name in ((0, "ours_crs"), (1, "ours_crs_unrolled")):
        st = torch.cuda.current_stream()

        def launch():
            _lib.check(slib.sellb_spmv_crs(rpt64.data_ptr(), col32.data_ptr(), valt.data_ptr(),
                                           code, x.data_ptr(), y.data_ptr(), 0, n, 0, unrolled,
                                           st.cuda_stream))
        for _ in range(10):
            launch()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(reps):
            launch()
        e1.record(st)
        e1.synchronize()
        rec(name, e0.elapsed_time(e1) / reps, y.cpu().numpy())
    del rpt64, col32, valt
    lib = ctypes.CDLL(LIB)
    # cuSPARSE CSR
    rpt = torch.from_numpy(m.rpt.astype(np.int32)).cuda()
    col = torch.from_numpy(m.col.astype(np.int32)).cuda()
    val = torch.from_numpy(val_h).cuda()
    y = torch.zeros(n, dtype=tdt, device="cuda")
    for fmt, name in ((0, "cusparse_csr_alg1"), (1, "cusparse_csr_alg2")):
        ms = csp(lib, fmt, f32, n, nc, nnz, nnz, rpt, col, val, x, y, reps)
        rec(name, ms, y.cpu().numpy())
    del rpt, col, val
    # cuSPARSE Sliced-ELL from our σ=1 layout, pads marked -1
    cs = s1.cs
    cl = s1.cl
    rl = s1.row_lengths
    slots = int(cs[-1])
    chunk = np.repeat(np.arange(s1.n_chunks, dtype=np.int64), cl.astype(np.int64) * 32)
    k = np.arange(slots, dtype=np.int64) - cs[chunk]
    pad = (k // 32) >= rl[chunk * 32 + k % 32]
    del chunk, k
    scol_h = s1.col.copy()
    scol_h[pad] = -1
    soff = torch.from_numpy(cs.astype(np.int32)).cuda()
    scol = torch.from_numpy(scol_h).cuda()
    sval = torch.from_numpy(s1.val.astype(dt)).cuda()
    del scol_h, pad
    y = torch.zeros(n, dtype=tdt, device="cuda")
    ms = csp(lib, 2, f32, n, nc, nnz, slots, soff, scol, sval, x, y, reps)
    rec("cusparse_sell32_alg1", ms, y.cpu().numpy())
    s1.free()
    return out


def main():
    args = [a for a in sys.argv[1:] if not a.startswith("--")]
    f32 = "--f32" in sys.argv
    build()
    for cfg in args or ["cfg1", "cfg2", "cfg3", "cfg4"]:
        reps = 200 if cfg in ("cfg1", "cfg2") else 50
        print(json.dumps(run(cfg, f32, reps)), flush=True)


if __name__ == "__main__":
    main()
