"""Matrix Market read/write throughput: native body parser / formatter vs the
reference-equivalent NumPy path (np.loadtxt / np.savetxt batches, io.py).
    python tools/mm_bench.py [n_entries]"""
import os
import sys
import tempfile
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb  # noqa: E402
from paper_1307_6209_b200 import mmio  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5_000_000
rng = np.random.default_rng(0)
N = max(1000, int(n ** 0.5) * 20)
m = sb.canonicalize_coo(sb.COOMatrix(N, N, rng.integers(0, N, n), rng.integers(0, N, n),
                                     rng.standard_normal(n)))
d = tempfile.mkdtemp()
p = os.path.join(d, "b.mtx")
t = time.perf_counter()
sb.write_matrix_market(m, p)
tw = time.perf_counter() - t
size = os.path.getsize(p)
t = time.perf_counter()
np.savetxt(os.path.join(d, "ref.txt"),
           np.column_stack((m.rows + 1, m.cols + 1, m.vals)), fmt="%d %d %.17g")
tw_ref = time.perf_counter() - t
t = time.perf_counter()
back = sb.read_matrix_market(p)
tr = time.perf_counter() - t
t = time.perf_counter()
body = mmio._slow_read(p, 3, 3, m.nnz)
tr_ref = time.perf_counter() - t
raw = open(p, "rb").read()
head = mmio._split_header(raw)
t = time.perf_counter()
fast = mmio._parse_body(raw, head[3], 3, m.nnz)
tp = time.perf_counter() - t
dev = None
try:
    import torch
    if torch.cuda.is_available():
        sb.read_matrix_market(p, device=0)          # warm-up (CUDA context, pool)
        t = time.perf_counter()
        back_d = sb.read_matrix_market(p, device=0)
        dev = time.perf_counter() - t
        assert np.array_equal(back_d.vals, m.vals)
except ImportError:
    pass
assert np.array_equal(back.vals, m.vals)
assert np.array_equal(body[:, 2], m.vals)
print(f"entries {m.nnz}  file {size / 1e6:.0f} MB  threads {os.cpu_count()}")
print(f"write: native {tw:.2f} s ({size / tw / 1e6:.0f} MB/s)   np.savetxt {tw_ref:.2f} s")
print(f"read:  native+canonicalise {tr:.2f} s ({size / tr / 1e6:.0f} MB/s)   "
      f"np.loadtxt body only {tr_ref:.2f} s ({size / tr_ref / 1e6:.0f} MB/s)")
print(f"       native body parse only {tp:.2f} s ({size / tp / 1e6:.0f} MB/s)"
      + (f"   read with device canonicalisation {dev:.2f} s ({size / dev / 1e6:.0f} MB/s)"
         if dev else ""))
