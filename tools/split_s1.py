"""sigma=1 layouts: a few SpMVs for an ncu launch list (long rows in a
separate kernel with SELLB_LONG_REST=1)."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
which = sys.argv[1]
if which == "cfg3":
    m = generate.powerlaw(4_000_000)
else:
    m = sb.coo_to_crs(sb.gen_skewed(1 << 21, 8, 2048, 1024))
s = sb.crs_to_sell(m, 32, 1)
x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
for _ in range(3):
    sb.spmv_sell(s, x, y)
torch.cuda.synchronize()
print("ok", s.variant)
