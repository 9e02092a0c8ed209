import sys, torch, numpy as np
sys.path.insert(0, '.')
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate, _lib
lib = _lib.load()
for lmax in (4096, 1024, 512, 256):
    m = generate.powerlaw(4_000_000, lmax=lmax)
    for mode in (True, False):
        s = sb.crs_to_sell(m, 32, 1)
        s.set_packed(mode)
        x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
        y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device='cuda')
        st = torch.cuda.current_stream().cuda_stream
        for _ in range(5): lib.sellb_spmv(s.handle, x.data_ptr(), y.data_ptr(), 0, s.n_chunks, 0, 0, st)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50): lib.sellb_spmv(s.handle, x.data_ptr(), y.data_ptr(), 0, s.n_chunks, 0, 0, st)
        e1.record(); e1.synchronize()
        ms = e0.elapsed_time(e1) / 50
        print(f"lmax {lmax} packed {mode}: nnz {m.nnz} {ms*1000:.1f} us {2*m.nnz/ms/1e6:.1f} GF/s", flush=True)
        s.free()
