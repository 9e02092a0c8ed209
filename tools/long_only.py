"""One matrix with only long rows (128 x 2048, sorted) for profiling the long-row role."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
m = sb.coo_to_crs(sb.gen_skewed(1 << 21, 1, 2048, 128))
s = sb.crs_to_sell(m, 32, 1 << 21)
x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
for _ in range(4):
    sb.spmv_sell(s, x, y)
torch.cuda.synchronize()
print("ok")
