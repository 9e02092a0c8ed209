"""Decompose cfg4 (skewed) kernel time: with/without spikes, long-row role on/off."""
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
    inf = s.info()
    return e0.elapsed_time(e1) / reps * 1e3, inf.nnz, inf.variant

for spikes in (1024, 0):
    m = sb.coo_to_crs(sb.gen_skewed(1 << 21, 8, 2048, spikes))
    for sigma in (1, 1 << 21):
        us, nnz, var = t(m, 32, sigma)
        print(f"spikes={spikes} sigma={sigma} LONG_TH={os.environ.get('SELLB_LONG_TH','256')}: {us:.1f} us  nnz={nnz} variant={var} -> {2*nnz/us/1e3:.0f} GF/s", flush=True)
