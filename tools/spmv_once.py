"""Build one config and run a few SpMVs (for ncu captures of one kernel):
python tools/spmv_once.py cfg3 SIGMA [reps]  (SELLB_* switches apply)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import _lib, generate

cfg, sigma = sys.argv[1], int(sys.argv[2])
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 3
f32 = len(sys.argv) > 4 and sys.argv[4] == "f32"
if cfg == "cfg3":
    m = generate.powerlaw(4_000_000)
elif cfg == "cfg4":
    from paper_1307_6209_b200 import coo_to_crs, gen_skewed
    m = coo_to_crs(gen_skewed(1 << 21, 8, 2048, 1024))
elif cfg == "cfg2":
    m = generate.stencil27(128)
else:
    m = generate.laplace2d(1000)
dt = np.float32 if f32 else np.float64
if f32:
    from paper_1307_6209_b200 import CRSMatrix
    m = CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val.astype(np.float32))
s = sb.crs_to_sell(m, 32, sigma, dtype=dt)
print("variant", s.variant, "packed", s.packed, "long", s.long_rows_info(), flush=True)
x = torch.from_numpy(generate.rhs(m.n_cols).astype(dt)).cuda()
y = torch.zeros(s.n_rows_padded, dtype=torch.float32 if f32 else torch.float64, device="cuda")
lib = _lib.load()
st = torch.cuda.current_stream().cuda_stream
for _ in range(reps):
    _lib.check(lib.sellb_spmv(s.handle, x.data_ptr(), y.data_ptr(), 0, s.n_chunks, 0, 0, st))
torch.cuda.synchronize()
print("done")
