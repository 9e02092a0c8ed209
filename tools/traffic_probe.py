"""One SpMV of a BASELINE layout, for an ncu DRAM-bytes reading.
    python tools/traffic_probe.py cfg3 512"""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
from bench import make_matrix
m, _ = make_matrix(sys.argv[1])
s = sb.crs_to_sell(m, 32, int(sys.argv[2]))
x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
for _ in range(3):
    sb.spmv_sell(s, x, y)
torch.cuda.synchronize()
print("ok")
