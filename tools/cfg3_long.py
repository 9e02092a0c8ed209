"""cfg3 sigma=N: a few SpMVs for an ncu launch list of the long-row kernels."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
sigma = int(sys.argv[1]) if len(sys.argv) > 1 else 4_000_000
m = generate.powerlaw(4_000_000)
s = sb.crs_to_sell(m, 32, sigma)
x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
for _ in range(3):
    sb.spmv_sell(s, x, y)
torch.cuda.synchronize()
print("ok", s.variant)
