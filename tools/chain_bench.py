"""Chained SpMVs in permuted space (spmv_chain, one CUDA graph) vs single
launches: per-product time and GF/s.  python tools/chain_bench.py [cfg] [steps]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb  # noqa: E402
from paper_1307_6209_b200 import generate  # noqa: E402
from bench import make_matrix  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "cfg2"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 200
m, desc = make_matrix(cfg)
sigma = 1 if cfg in ("cfg1", "cfg2") else m.n_rows
m = sb.CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val * (1.0 / 64))   # bounded powers
s = sb.crs_to_sell(m, 32, sigma, permute_cols=True)
x = torch.from_numpy(sb.permute_vector(generate.rhs(m.n_cols), s.perm)).cuda()
flops = 2.0 * m.nnz
for graph in (True, False):
    ch = sb.SpmvChain(s, steps, graph=graph)
    ch.run(x)                                    # capture / warm-up
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        ch.run(x)
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / (3 * steps)
    # one product on its own, same layout, back to back
    y = torch.empty(s.n_rows_padded, dtype=x.dtype, device="cuda")
    xx = torch.zeros(s.n_rows_padded, dtype=x.dtype, device="cuda")
    xx[:m.n_rows] = x
    for _ in range(5):
        sb.spmv_sell(s, xx[:m.n_rows], y)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(steps):
        sb.spmv_sell(s, xx[:m.n_rows], y)
    e1.record()
    e1.synchronize()
    ms1 = e0.elapsed_time(e1) / steps
    print(f"{desc}, permuted SELL-32-{sigma}: {steps} chained products "
          f"({'graph' if graph else 'launches'}) {ms * 1e3:.1f} us each, "
          f"{flops / ms / 1e6:.1f} GF/s; same x every launch {ms1 * 1e3:.1f} us, "
          f"{flops / ms1 / 1e6:.1f} GF/s", flush=True)
