"""Run the device CRS kernel a few times on one config (ncu captures)."""
import sys
import numpy as np
import torch
sys.path.insert(0, ".")
from paper_1307_6209_b200 import _lib, generate
from bench import make_matrix
m, _ = make_matrix(sys.argv[1])
unrolled = int(sys.argv[2]) if len(sys.argv) > 2 else 0
t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
     for k, v in (("rpt", m.rpt), ("col", m.col), ("val", m.val), ("x", generate.rhs(m.n_cols)))}
y = torch.zeros(m.n_rows, dtype=torch.float64, device="cuda")
lib = _lib.load()
for _ in range(3):
    _lib.check(lib.sellb_spmv_crs(t["rpt"].data_ptr(), t["col"].data_ptr(), t["val"].data_ptr(),
                                  0, t["x"].data_ptr(), y.data_ptr(), 0, m.n_rows, 0, unrolled,
                                  torch.cuda.current_stream().cuda_stream))
torch.cuda.synchronize()
print("done")
