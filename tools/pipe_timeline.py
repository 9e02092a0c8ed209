"""Timeline of the pipelined host path, emulated with torch streams + events."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import _lib, generate

m = generate.stencil27(128)
s = sb.crs_to_sell(m, 32, 1)
lib = _lib.load()
n, npad, nch = m.n_cols, s.n_rows_padded, s.n_chunks
xh = torch.from_numpy(generate.rhs(n)).pin_memory()
yh = torch.empty(npad, dtype=torch.float64).pin_memory()
xd = torch.empty(n, dtype=torch.float64, device="cuda")
yd = torch.empty(npad, dtype=torch.float64, device="cuda")
P = int(sys.argv[1]) if len(sys.argv) > 1 else 16
s1, s2, s3 = torch.cuda.Stream(), torch.cuda.Stream(), torch.cuda.Stream()
xo = [n * i // P for i in range(P + 1)]
bc = [nch * i // P for i in range(P + 1)]


def run(record):
    t = {}
    e0 = torch.cuda.Event(enable_timing=True)
    e0.record(torch.cuda.current_stream())
    s1.wait_event(e0)
    s2.wait_event(e0)
    ex = []
    for i in range(P):
        with torch.cuda.stream(s1):
            xd[xo[i]:xo[i + 1]].copy_(xh[xo[i]:xo[i + 1]], non_blocking=True)
            e = torch.cuda.Event(enable_timing=True)
            e.record(s1)
            ex.append(e)
    eb = []
    for b in range(P):
        need = min(b + 1, P - 1)
        s2.wait_event(ex[need])
        _lib.check(lib.sellb_spmv(s.handle, xd.data_ptr(), yd.data_ptr(), bc[b], bc[b + 1], 0, 0,
                                  s2.cuda_stream))
        e = torch.cuda.Event(enable_timing=True)
        e.record(s2)
        eb.append(e)
        s3.wait_event(e)
        with torch.cuda.stream(s3):
            r0, r1 = bc[b] * 32, bc[b + 1] * 32
            yh[r0:r1].copy_(yd[r0:r1], non_blocking=True)
    ed = torch.cuda.Event(enable_timing=True)
    ed.record(s3)
    torch.cuda.synchronize()
    if record:
        print("x pieces done (ms):", " ".join(f"{e0.elapsed_time(e):.3f}" for e in ex))
        print("blocks done   (ms):", " ".join(f"{e0.elapsed_time(e):.3f}" for e in eb))
        print("all done      (ms):", f"{e0.elapsed_time(ed):.3f}")


for _ in range(5):
    run(False)
run(True)
t0 = time.perf_counter()
for _ in range(100):
    run(False)
print(f"P={P}: {(time.perf_counter() - t0) / 100 * 1e3:.3f} ms/step wall")
