import os, sys, torch
sys.path.insert(0, "/root/repo")
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
m = sb.coo_to_crs(sb.gen_skewed(1 << 16, 8, 2048, int(sys.argv[1]) if len(sys.argv) > 1 else 64))
s = sb.crs_to_sell(m, 32, 1 << 16)
x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
y = sb.spmv_sell(s, x)
torch.cuda.synchronize()
print("ok")
