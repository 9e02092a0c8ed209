"""cfg4 σ=N split: full matrix vs its bulk (no spikes) vs its spikes alone
(base 1), one SELL-32-N build each, region-timed back-to-back launches."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate


def t(m, C=32, sigma=1 << 21, reps=100):
    s = sb.crs_to_sell(m, C, sigma)
    x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
    y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
    for _ in range(5):
        sb.spmv_sell(s, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        sb.spmv_sell(s, x, y)
    e1.record()
    e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, s.variant


n = 1 << 21
for name, base, spl, cnt in (("full", 8, 2048, 1024), ("bulk", 8, 2048, 0),
                             ("spikes", 1, 2048, 1024), ("spikes_512x4096", 1, 4096, 512)):
    m = sb.coo_to_crs(sb.gen_skewed(n, base, spl, cnt))
    for sigma in ((1 << 21, 1) if name == "full" else (1 << 21,)):
        us, var = t(m, sigma=sigma)
        print(f"{name:16} s={sigma:<8} nnz={m.nnz:>9} {us:7.1f} us {var} "
              f"{m.nnz * 12 / us / 1e3:7.1f} GB/s(matrix)", flush=True)
