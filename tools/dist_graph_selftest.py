"""DistSpmv.capture with real NCCL traffic on one GPU: a world-1 DistSpmv
whose halo plan sends a scattered set of x entries to itself (gather kernel
-> NCCL self send/recv -> scatter kernel), so the captured step holds NCCL
P2P kernels next to the library's.  The replayed graph must reproduce the
eager y bitwise, then follow a new x.  Run under torchrun --nproc-per-node 1;
prints 'dist graph selftest ok'."""
import os
import sys

import numpy as np
import torch
import torch.distributed as tdist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_6209_b200 import generate                       # noqa: E402
from paper_1307_6209_b200.dist import HaloPlan, cuda_engine_factory, setup  # noqa: E402

dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
tdist.init_process_group("nccl", device_id=dev)
crs = generate.stencil27(32)
n = crs.n_rows
bounds = np.array([0, n], dtype=np.int64)
idx = np.arange(0, n, 3, dtype=np.int32)           # scattered: gather/scatter path
plan = HaloPlan(0, 1, bounds, recv={0: idx}, send={0: idx}, need_x0={0: False})
ds = setup(crs, bounds, 32, 1, 0, 1, dev, cuda_engine_factory(32, 1, dev), plan=plan)
assert ds.send_ops and ds.recv_ops and ds.send_ops[0][2] is not None
x = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, n)).to(dev)
ds.x_local.copy_(x)
print("setup done", flush=True)
y_eager = ds.step().clone()
torch.cuda.synchronize()
print("eager done", flush=True)
assert ds.capture(), "graph not kept"
print("capture done", flush=True)
assert ds.graph_launches >= 3, ds.graph_launches       # gather, spmv, scatter
y_graph = ds.step().clone()
print("replay done", flush=True)
assert torch.equal(y_graph.view(torch.int64), y_eager.view(torch.int64))
x2 = torch.from_numpy(np.random.default_rng(6).uniform(-1, 1, n)).to(dev)
ds.x_local.copy_(x2)
y2 = ds.step().clone()
ds.graph, g = None, ds.graph
y2_eager = ds.step().clone()
ds.graph = g
del g       # the only reference must be ds.graph for release() to free it
print("eager-after-graph done", flush=True)
assert torch.equal(y2.view(torch.int64), y2_eager.view(torch.int64))
ds.release()
torch.cuda.synchronize()
tdist.destroy_process_group()
print("dist graph selftest ok", flush=True)
