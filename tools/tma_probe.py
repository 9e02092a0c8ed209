"""A/B of the TMA bulk-copy SpMV path (SELLB_TMA=1) vs the LDG kernel, with
bitwise check against the default path."""
import os
import subprocess
import sys

if len(sys.argv) > 1 and sys.argv[1] == "child":
    import numpy as np
    import torch
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import generate
    for name, mk, dt in (("cfg2", lambda: generate.stencil27(128), np.float64),
                         ("cfg2_f32", lambda: generate.stencil27(128), np.float32),
                         ("cfg5_s512_2^24", lambda: None, np.float64)):
        if name.startswith("cfg5"):
            rpt, col, val = generate.hamiltonian_device(1 << 24)
            s = sb.crs_to_sell_device(rpt, col, val, 1 << 24, 1 << 24, 32, 512)
            nc = 1 << 24
        else:
            m = mk()
            s = sb.crs_to_sell(m, 32, 1, dtype=dt)
            nc = m.n_cols
        tdt = torch.float32 if dt == np.float32 else torch.float64
        x = torch.from_numpy(generate.rhs(nc, dtype=dt)).cuda()
        y = torch.zeros(s.n_rows_padded, dtype=tdt, device="cuda")
        for _ in range(10):
            sb.spmv_sell(s, x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(200):
            sb.spmv_sell(s, x, y)
        e1.record(); e1.synchronize()
        t = e0.elapsed_time(e1) / 200 / 1e3
        out = os.environ.get("OUT")
        np.save(f"{out}_{name}.npy", y.cpu().numpy())
        print(f"TMA={os.environ.get('SELLB_TMA', '0')} {name}: {t*1e6:.1f} us {2*s.nnz/t/1e9:.1f} GF/s", flush=True)
else:
    import numpy as np
    os.makedirs("gpurun_out", exist_ok=True)
    for tma, u in (("0", "16"), ("1", "8"), ("1", "16"), ("1", "32")):
        subprocess.run([sys.executable, __file__, "child"],
                       env={**os.environ, "SELLB_TMA": tma, "SELLB_TMA_U": u,
                            "OUT": f"gpurun_out/tma{tma}_{u}"}, timeout=600)
        print("  U =", u, flush=True)
    for u in ("8", "16", "32"):
        for name in ("cfg2", "cfg2_f32", "cfg5_s512_2^24"):
            a = np.load(f"gpurun_out/tma0_16_{name}.npy")
            b = np.load(f"gpurun_out/tma1_{u}_{name}.npy")
            print(u, name, "bitwise equal:", a.tobytes() == b.tobytes())
