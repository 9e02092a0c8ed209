"""Time the host-array SpMV path (sellb_spmv_host) with pinned buffers for
several pipeline depths (SELLB_PIPE) and the serial path."""
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
    print(os.environ.get("SELLB_PIPE", "-"), os.environ.get("SELLB_NO_PIPELINE", "-"),
          f"{(time.perf_counter() - t0) / 200 * 1e3:.3f} ms/step", flush=True)
else:
    for env in ({"SELLB_NO_PIPELINE": "1"}, {"SELLB_PIPE": "2"}, {"SELLB_PIPE": "4"},
                {"SELLB_PIPE": "8"}, {"SELLB_PIPE": "16"}):
        subprocess.run([sys.executable, __file__, "child"], env={**os.environ, **env})
