"""Time the long-row role in isolation: skewed matrices whose bulk is tiny."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate

def t(m, C, sigma, reps=50):
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
    e1.record(); e1.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3, s.info().n_long if hasattr(s.info(), "n_long") else None

for base, spikes, spike_len in ((1, 1024, 2048), (8, 1024, 2048), (1, 128, 2048), (1, 1024, 512), (1, 1024, 8192)):
    m = sb.coo_to_crs(sb.gen_skewed(1 << 21, base, spike_len, spikes))
    for sigma in (1, 1 << 21):
        us, _ = t(m, 32, sigma)
        print(f"base={base} spikes={spikes}x{spike_len} sigma={sigma}: {us:.1f} us", flush=True)
