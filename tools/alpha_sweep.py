#!/usr/bin/env python3
"""sigma sweep with the performance model fed by MEASURED DRAM bytes -- the
B200 analog of the reference's `sellkit sweep-sigma` (cli.py:296-320), which
simulates alpha with an LRU model (cachesim.py:49-75).  Here alpha comes from
ncu's dram__bytes_read.sum + dram__bytes_write.sum of the SpMV kernel.

Each layout is measured as built (SELLB shadow dropped) and, where the
build's cost model adds the SELL-32-N shadow execution layout, once more with
it -- the first row is the paper's sigma effect, the second
what spmv_sell runs by default.

On the GPU box (one ncu pass over the profiled SpMVs only -- the run brackets
each with cudaProfilerStart/Stop and records how many kernels it launched):
    ncu --metrics dram__bytes_read.sum,dram__bytes_write.sum,gpu__time_duration.sum \
        --profile-from-start off --csv --log-file gpurun_out/alpha.csv \
        python tools/alpha_sweep.py run gpurun_out/alpha_layouts.json
and without ncu for timing:
    python tools/alpha_sweep.py time gpurun_out/alpha_times.json
Here (CPU):
    python tools/alpha_sweep.py traffic gpurun_out/alpha_layouts.json \
        gpurun_out/alpha.csv profiles/ncu_traffic.json
    python tools/alpha_sweep.py report gpurun_out/alpha_layouts.json \
        gpurun_out/alpha.csv gpurun_out/alpha_times.json > profiles/r01_alpha_sweep.md
"""
import csv
import io
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

LAYOUTS = [("cfg2", 1)] + [("cfg3", s) for s in (1, 32, 64, 128, 256, 512, 1024, 4096,
                                                  4_000_000)]


def matrices():
    from paper_1307_6209_b200 import generate
    cache = {}
    for name, sigma in LAYOUTS:
        if name not in cache:
            cache[name] = generate.stencil27(128) if name == "cfg2" else generate.powerlaw()
        yield name, sigma, cache[name]


def run(out_json, timed=False):

    import torch
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import _lib, generate
    lib = _lib.load()
    rows = []
    for name, sigma, m in matrices():
        s = sb.crs_to_sell(m, 32, sigma)
        auto_shadow = s.shadow
        x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
        y = torch.zeros(s.n_rows_padded, dtype=torch.float64, device="cuda")
        for mode in ((False, None) if auto_shadow else (False,)):
            s.set_shadow(mode)
            rows.append(measure(sb, lib, torch, name, sigma, s, x, y, timed))
        s.free()
    json.dump(rows, open(out_json, "w"), indent=1)


def measure(sb, lib, torch, name, sigma, s, x, y, timed):
    info = s.info()
    be, vs, cs = s.sector_occupancy()
    rl = s.row_lengths
    # 64-byte granularity (two sectors): 8 fp64 lanes of val, 16 of col
    v64 = int(rl.reshape(-1, 8).max(1).sum()) * 2
    c64 = int(rl.reshape(-1, 16).max(1).sum()) * 2
    mb32, mb64, mx = s.streamed_bytes()
    rec = {"name": name, "sigma": sigma, "nnz": info.nnz, "n_rows": info.n_rows,
           "stream32": mb32, "stream64": mb64, "stream_extra": mx,
           "long_rows": s.long_rows_info(),
           "n_cols": info.n_cols, "n_pad": info.n_rows_padded, "n_chunks": info.n_chunks,
           "slots": info.slots, "beta": info.nnz / info.slots, "beta_eff": be,
           "val_sectors": vs, "col_sectors": cs, "val_sectors64": v64,
           "col_sectors64": c64, "shadow": s.shadow,
           "variant": ("shadow SELL-32-%s" % ("N" if s.shadow_sigma >= info.n_rows_padded
                                               else s.shadow_sigma)
                       if s.shadow else s.variant + ("+packed" if s.packed else ""))}
    sb.spmv_sell(s, x, y)                # warm (first-use setup outside the profiled range)
    torch.cuda.synchronize()
    if timed:
        for _ in range(5):
            sb.spmv_sell(s, x, y)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(50):
            sb.spmv_sell(s, x, y)
        e1.record()
        e1.synchronize()
        rec["kernel_s"] = e0.elapsed_time(e1) / 50 / 1e3
    else:
        n0 = lib.sellb_launch_count()
        torch.cuda.profiler.start()
        sb.spmv_sell(s, x, y)            # the one profiled SpMV
        torch.cuda.synchronize()
        torch.cuda.profiler.stop()
        rec["launches"] = int(lib.sellb_launch_count() - n0)
    return rec


def dram_per_layout(layouts_json, ncu_csv):
    """[(row, dram bytes of that layout's one SpMV)] from the run's layouts
    and the ncu CSV (a layout's launches summed)."""
    rows = json.load(open(layouts_json))
    lines = open(ncu_csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    recs = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    per = {}
    for r in recs:
        if r["Metric Name"] in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            per[r["ID"]] = per.get(r["ID"], 0.0) + float(r["Metric Value"]) * scale[r["Metric Unit"]]
    ids = sorted(per, key=int)
    out, k = [], 0
    for row in rows:
        n = row.get("launches", 1)
        out.append((row, sum(per[i] for i in ids[k:k + n])))
        k += n
    assert k == len(ids), (k, len(ids))
    return out


def traffic(layouts_json, ncu_csv, traffic_json):
    """Merge the measured DRAM bytes into profiles/ncu_traffic.json (the keys
    bench.py reads: <cfg>_s<sigma>_f64[_shadow])."""
    d = json.load(open(traffic_json))
    for row, dram in dram_per_layout(layouts_json, ncu_csv):
        key = f"{row['name']}_s{row['sigma']}_f64" + ("_shadow" if row.get("shadow") else "")
        d[key] = int(dram)
    json.dump(d, open(traffic_json, "w"), indent=1)


def report(layouts_json, ncu_csv, times_json):
    from paper_1307_6209_b200 import model
    rows = json.load(open(layouts_json))
    times = {(r["name"], r["sigma"], r.get("shadow", False)): r["kernel_s"]
             for r in json.load(open(times_json))}
    lines = open(ncu_csv).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    recs = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    per = {}
    for r in recs:
        per.setdefault(r["ID"], {})[r["Metric Name"]] = (float(r["Metric Value"]),
                                                         r["Metric Unit"])
    ids = sorted(per, key=int)
    # one SpMV may be two launches (the packed copy's row-run kernel plus the
    # warp-per-row kernel for its long rows): sum the DRAM bytes of each
    # layout's launches
    def n_launch(row):
        if "launches" in row:                    # counted by the library during the run
            return row["launches"]
        packed = "+packed" in row["variant"]
        return 2 if packed and row["long_rows"]["n_long"] > 0 else 1
    groups, k = [], 0
    for row in rows:
        n = n_launch(row)
        groups.append(ids[k:k + n])
        k += n
    assert k == len(ids), (k, len(ids))
    merged = {}
    for g in groups:
        acc = {}
        for i in g:
            for name, (v, u) in per[i].items():
                f = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u)
                if f is None:
                    acc.setdefault(name, (v, u))
                    continue
                prev = acc.get(name, (0.0, "byte"))[0]
                acc[name] = (prev + v * f, "byte")
        merged[g[0]] = acc
    per = merged
    ids = [g[0] for g in groups]
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(
        os.path.abspath(__file__))), "MEASURED_PEAKS.json")))["hbm_gbs"]
    print("# sigma sweep with measured alpha (one B200)\n")
    print("alpha_paper = `infer_alpha(dram, nnz, beta, N_nzr, line=32)` (model.py:124-142 "
          "with B200's 32 B sector as the line); alpha_eff = `alpha_from_traffic` with the "
          "bytes the kernels actually stream as configured (`sellb_streamed_bytes`: all slots "
          "of pad-incl chunks, touched 32 B / 64 B sectors of bulk rows + row_lengths for "
          "pad-skip chunks, long rows from the contiguous side table).  Ideal alpha = 1/N_nzc.  DRAM = ncu "
          "dram__bytes_read.sum + dram__bytes_write.sum of one cold SpMV launch; "
          "GF/s from CUDA events (50 warm launches).  Rows marked `shadow` are the same "
          "layout executed through its SELL-32 shadow copy (spmv_sell's default for "
          "irregular layouts, bit-identical y); beta / beta_eff there are the CALLER's "
          "layout; matrix MB and alpha_eff use the bytes the shadow streams.\n")
    print("| matrix | sigma | beta | beta_eff | variant | DRAM MB | V_alg MB | matrix MB (32 B / 64 B) | "
          "alpha_paper | in range | alpha_eff 32 B | alpha_eff 64 B | ideal alpha | "
          "B paper (ideal alpha) | GF/s | paper P = b/B GF/s |")
    print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
    for i, row in zip(ids, rows):
        d = per[i]
        rd = d["dram__bytes_read.sum"][0] * scale[d["dram__bytes_read.sum"][1]]
        wr = d["dram__bytes_write.sum"][0] * scale[d["dram__bytes_write.sum"][1]]
        dram = rd + wr
        nnz, n = row["nnz"], row["n_rows"]
        nzr, nzc = nnz / n, nnz / row["n_cols"]
        a_p = model.infer_alpha(dram, nnz, row["beta"], nzr, line_bytes=32)
        # what the kernels stream as configured (sellb_streamed_bytes: bulk
        # sectors, long rows from the side table, row_lengths)
        mat, mat64, extra = row["stream32"], row["stream64"], row["stream_extra"]
        a_e = model.alpha_from_traffic(dram, nnz, mat, row["n_pad"], row["n_chunks"],
                                       extra_bytes=extra)
        a_64 = model.alpha_from_traffic(dram, nnz, mat64, row["n_pad"], row["n_chunks"],
                                        extra_bytes=extra)
        v_alg = model.algorithmic_bytes(nnz, row["n_cols"], row["n_pad"], row["n_chunks"])
        bal = model.code_balance_sell(1.0 / nzc, row["beta"], nzr)
        # the timed run builds its own layouts; its shadow choice is timed too
        t = times.get((row["name"], row["sigma"], row.get("shadow", False)))
        gfs = f"{2 * nnz / t / 1e9:.1f}" if t else "n/a"
        print(f"| {row['name']} | {row['sigma']} | {row['beta']:.4f} | {row['beta_eff']:.4f} | "
              f"{row['variant']} | {dram / 1e6:.1f} | {v_alg / 1e6:.1f} | "
              f"{mat / 1e6:.0f} / {mat64 / 1e6:.0f} | {a_p.alpha:.3f} | "
              f"{a_p.in_range} | {a_e.alpha:.3f} | {a_64.alpha:.3f} | {1 / nzc:.3f} | {bal:.3f} | "
              f"{gfs} | {peak / bal:.1f} |")


if __name__ == "__main__":
    if sys.argv[1] == "run":
        run(sys.argv[2])
    elif sys.argv[1] == "time":
        run(sys.argv[2], timed=True)
    elif sys.argv[1] == "traffic":
        traffic(sys.argv[2], sys.argv[3], sys.argv[4])
    else:
        report(sys.argv[2], sys.argv[3], sys.argv[4])
