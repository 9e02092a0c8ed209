#!/usr/bin/env python3
"""Markdown table of a tools/sweep.sh run:  python tools/sweep_table.py DIR > OUT.md"""
import glob
import json
import os
import sys

d0 = sys.argv[1]
rows = []
for f in sorted(glob.glob(os.path.join(d0, "*.json"))):
    try:
        d = json.loads(open(f).read().strip().splitlines()[-1])
    except (ValueError, IndexError):
        continue
    c, r = d["config"], d["roofline"]
    cpu = d.get("cpu_baseline") or {}
    rows.append((os.path.basename(f)[:-5], c["workload"], d["dtype"], c["beta"],
                 c["kernel_variant"], r["kernel_ms"], d["value"], r["achieved"], r["frac"],
                 c["parity_vs_oracle"], d["e2e"]["value"], cpu.get("value"),
                 (d.get("clocks") or {}).get("sm_mhz")))
print("# Config sweep (one B200, `sh tools/sweep.sh`)\n")
print("GF/s = 2·nnz/t (padding excluded); GB/s = algorithmic bytes / kernel time; frac of "
      "MEASURED_PEAKS hbm_gbs 6449.1 GB/s (measured copy). parity = device arrays and y "
      "bit-exact vs the oracle (cfg5: three 65536-row blocks). ref CPU = the reference's "
      "compiled core (oracle/_ref) on the box's 16 host threads, bounded sample.\n")
print("| run | workload | dtype | β | variant | kernel ms | GF/s | GB/s (alg) | frac | parity "
      "| e2e GF/s | ref CPU GF/s | SM MHz |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print("| " + " | ".join(str(v) for v in r) + " |")
