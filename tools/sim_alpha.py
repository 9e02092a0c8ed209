#!/usr/bin/env python3
"""Simulated alpha (LRU replay of the x stream, cachesim.py:49-75) beside the
measured one (profiles/r01_alpha_sweep.md) -- the comparison of the
reference's `sellkit sweep-sigma` (cli.py:296-320), with the replay on the
GPU (sellb_lru_stream_misses).

    python tools/sim_alpha.py gpurun_out/sim_alpha.json      (GPU box)
    python tools/sim_alpha.py report gpurun_out/sim_alpha.json > profiles/r01_sim_alpha.md
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LAYOUTS = [("cfg1", 1), ("cfg2", 1), ("cfg3", 1), ("cfg3", 128), ("cfg3", 512),
           ("cfg3", 4_000_000)]


def run(out):
    import torch
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import cachesim, generate
    l2 = torch.cuda.get_device_properties(0).L2_cache_size
    caches = [(l2 // 64) * 64, (l2 // 4 // 64) * 64, (l2 // 16 // 64) * 64, 1 << 20]
    mats = {}
    rows = []
    for name, sigma in LAYOUTS:
        if name not in mats:
            mats[name] = {"cfg1": lambda: generate.laplace2d(1000),
                          "cfg2": lambda: generate.stencil27(128),
                          "cfg3": generate.powerlaw}[name]()
        m = mats[name]
        s = sb.crs_to_sell(m, 32, sigma)
        n_nzr = s.nnz / s.n_rows_padded
        beta = sb.chunk_occupancy(s)
        for line in (32, 64):
            n_slots = (max(s.n_cols, 1) - 1) // (line // 8) + 1
            for cache in caches:
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                v = cachesim.simulate_rhs_traffic(s, cache, line)
                t_sim = time.perf_counter() - t0
                misses = (v - 12 * s.stored_slots - 16 * s.n_rows_padded) // line
                est = sb.infer_alpha(v, s.nnz, beta, n_nzr, line)
                rows.append({"name": name, "sigma": sigma, "line": line, "cache": cache,
                             "n_access": int(s.nnz), "n_lines": int(n_slots),
                             "misses": int(misses), "traffic": int(v), "beta": beta,
                             "alpha_paper": est.alpha, "in_range": bool(est.in_range),
                             "alpha_x": misses * line / (8.0 * s.nnz),
                             "ideal": s.n_cols / s.nnz, "t_sim_s": t_sim})
                print(json.dumps(rows[-1]), flush=True)
        del s
    with open(out, "w") as f:
        json.dump({"l2_bytes": l2, "rows": rows}, f, indent=1)


def report(path):
    d = json.load(open(path))
    print("# Simulated alpha (GPU LRU replay) vs measured\n")
    print(f"`tools/sim_alpha.py`, one B200 (L2 = {d['l2_bytes'] / 2**20:.1f} MiB).  "
          "alpha_x = x-line misses x line / (8 nnz): the x traffic per entry in "
          "units of one fp64 load (ideal = 1/N_nzc); alpha (paper) = `infer_alpha` on "
          "the simulated total with the format beta (cli.py:296-320).  Measured "
          "alpha_eff: `profiles/r01_alpha_sweep.md`.\n")
    print("| matrix | σ | line B | cache | accesses | misses | alpha_x | ideal 1/N_nzc "
          "| alpha (paper) | replay s |")
    print("|---|---|---|---|---|---|---|---|---|---|")
    for r in d["rows"]:
        c = r["cache"]
        cs = f"{c / 2**20:.1f} MiB"
        sig = "N" if r["sigma"] >= 1_000_000 else r["sigma"]
        print(f"| {r['name']} | {sig} | {r['line']} | {cs} | {r['n_access']:,} | "
              f"{r['misses']:,} | {r['alpha_x']:.4f} | {r['ideal']:.4f} | "
              f"{r['alpha_paper']:.3f} | {r['t_sim_s']:.2f} |")


if __name__ == "__main__":
    if sys.argv[1] == "report":
        report(sys.argv[2])
    else:
        run(sys.argv[1])
