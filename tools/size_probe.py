"""Attainable read bandwidth vs working-set size with a cold (flushed) L2:
our read-reduce kernel (membench) over buffers of 16 MB .. 2 GB, flushed
before every launch like bench.py does for small configs."""
import os
import sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1307_6209_b200 import _lib

lib = _lib.load()
l2 = torch.cuda.get_device_properties(0).L2_cache_size
flush = torch.empty(4 * l2, dtype=torch.uint8, device="cuda")
st = torch.cuda.current_stream().cuda_stream
for mb in (16, 38, 76, 152, 304, 703, 2048):
    n = mb * (1 << 20) // 8
    a = torch.rand(n, dtype=torch.float64, device="cuda")
    ts = []
    for i in range(30):
        lib.sellb_l2_flush(flush.data_ptr(), flush.numel(), st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        lib.sellb_read_sum(a.data_ptr(), n, None, st)
        e1.record()
        e1.synchronize()
        if i >= 5:
            ts.append(e0.elapsed_time(e1) / 1e3)
    t = sorted(ts)[len(ts) // 2]
    print(f"{mb:5d} MB cold read: {t*1e6:8.1f} us  {8*n/t/1e9:7.0f} GB/s")
