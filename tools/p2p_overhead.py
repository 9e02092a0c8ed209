"""Host-side cost of one DistSpmv-style exchange post (batch_isend_irecv of
a few P2P ops) under NCCL, measured at world size 1 with self send/recv --
the per-step CPU time the N>1 bench leg spends before the GPU work it
launches (run under torchrun --nproc-per-node 1)."""
import os
import time

import torch
import torch.distributed as tdist

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tdist.init_process_group("nccl", device_id=dev)
a = torch.zeros(16384, dtype=torch.float64, device=dev)
b = torch.zeros(16384, dtype=torch.float64, device=dev)
c = torch.zeros(1, dtype=torch.float64, device=dev)
d = torch.zeros(1, dtype=torch.float64, device=dev)
for nops in (2, 4, 6):
    def post():
        ops = []
        for i in range(nops // 2):
            ops.append(tdist.P2POp(tdist.isend, a if i == 0 else c, 0))
            ops.append(tdist.P2POp(tdist.irecv, b if i == 0 else d, 0))
        ws = tdist.batch_isend_irecv(ops)
        for w in ws:
            w.wait()
    for _ in range(50):
        post()
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        post()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"ops={nops}: host {1e6 * (t1 - t0) / n:.1f} us/post, "
          f"incl. drain {1e6 * (t2 - t0) / n:.1f} us/post", flush=True)
tdist.destroy_process_group()
