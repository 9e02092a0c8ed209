"""Very short chunks (1-3 nnz per row): default one-thread-per-row grid vs the
persistent warp sweep (SELLB_SWEEP=1), region-timed, 16M rows."""
import os
import sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate

n = 1 << 24
for w in (1, 2, 3):
    offs = np.arange(w) - (w // 2)
    rows = np.repeat(np.arange(n, dtype=np.int64), w)
    cols = rows + np.tile(offs, n)
    ok = (cols >= 0) & (cols < n)
    rows, cols = rows[ok], cols[ok]
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rpt[1:])
    m = sb.CRSMatrix(n, n, rpt, cols.astype(np.int32), np.full(len(cols), 0.5))
    s = sb.crs_to_sell(m, 32, 1)
    x = torch.from_numpy(generate.rhs(n)).cuda()
    y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
    for _ in range(5):
        sb.spmv_sell(s, x, y)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(50):
        sb.spmv_sell(s, x, y)
    e1.record()
    e1.synchronize()
    us = e0.elapsed_time(e1) / 50 * 1e3
    v = m.nnz * 12 + 16 * n
    print(f"w={w} {s.variant}: {us:.1f} us  {2 * m.nnz / us / 1e3:.0f} GF/s  "
          f"{v / us / 1e3:.0f} GB/s alg", flush=True)
