"""Time the host-array SpMV path (sellb_spmv_host) with pinned buffers for
several pipeline settings (env) and the serial path."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import time
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import _lib, generate
    m = generate.stencil27(128)
    s = sb.crs_to_sell(m, 32, 1)
    lib = _lib.load()
    xh = torch.from_numpy(generate.rhs(m.n_cols)).pin_memory()
    yh = torch.empty(s.n_rows_padded, dtype=torch.float64).pin_memory()
    for _ in range(5):
        _lib.check(lib.sellb_spmv_host(s.handle, xh.data_ptr(), yh.data_ptr(), 0, s.n_chunks, 0, 0, None))
    t0 = time.perf_counter()
    for _ in range(200):
        _lib.check(lib.sellb_spmv_host(s.handle, xh.data_ptr(), yh.data_ptr(), 0, s.n_chunks, 0, 0, None))
    dt = (time.perf_counter() - t0) / 200
    ok = yh.numpy().tobytes() == sb.spmv_sell(s, torch.from_numpy(generate.rhs(m.n_cols)).cuda()).cpu().numpy().tobytes()
    tag = " ".join(f"{k}={v}" for k, v in os.environ.items() if k.startswith("SELLB_"))
    print(f"[{tag}] {dt*1e3:.3f} ms/step  {2*s.nnz/dt/1e9:.1f} GF/s  exact={ok}", flush=True)
else:
    for env in ({"SELLB_NO_PIPELINE": "1"}, {"SELLB_PIPE": "4", "SELLB_PIPE_RAMP": "0"},
                {"SELLB_PIPE": "4"}, {"SELLB_PIPE": "5"}, {"SELLB_PIPE": "6"},
                {"SELLB_PIPE": "7"}, {"SELLB_PIPE": "5", "SELLB_NO_ZEROCOPY": "1"}):
        subprocess.run([sys.executable, __file__, "child"], env={**os.environ, **env})
