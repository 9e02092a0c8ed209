import sys, numpy as np, torch
sys.path.insert(0, '.')
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate, _lib
n = int(sys.argv[1])
rpt, col, val = generate.hamiltonian_device(n, device=0)
s = sb.crs_to_sell_device(rpt, col, val, n, n, 32, 512)
x = np.random.default_rng(12345).uniform(-1, 1, n)
xd = torch.from_numpy(x).cuda(); yd = torch.zeros(s.n_rows_padded, dtype=torch.float64, device='cuda')
_lib.check(_lib.load().sellb_spmv(s.handle, xd.data_ptr(), yd.data_ptr(), 0, s.n_chunks, 0, 0, torch.cuda.current_stream().cuda_stream))
yr = yd.cpu().numpy()
for it in range(4):
    y = np.full(s.n_rows_padded, np.nan)
    sb.spmv_sell(s, x, y)
    bad = np.nonzero(y.view(np.int64) != yr.view(np.int64))[0]
    print(it, len(bad), bad[:5], bad[-5:] if len(bad) else '', flush=True)
    if len(bad):
        print('  y', y[bad[:3]], 'ref', yr[bad[:3]])
# variants: pinned x (torch), pageable y; pageable x, pinned y
xp = torch.from_numpy(x).pin_memory().numpy()
y = np.full(s.n_rows_padded, np.nan)
sb.spmv_sell(s, xp, y); print('pinned x', int((y.view(np.int64) != yr.view(np.int64)).sum()))
yp = torch.full((s.n_rows_padded,), float('nan'), dtype=torch.float64).pin_memory().numpy()
sb.spmv_sell(s, x, yp); print('pinned y', int((yp.view(np.int64) != yr.view(np.int64)).sum()))
sb.spmv_sell(s, xp, yp); print('both pinned', int((yp.view(np.int64) != yr.view(np.int64)).sum()))
