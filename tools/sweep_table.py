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
    c, r, det = d["config"], d["roofline"], d["details"]
    cpu = d.get("cpu_baseline") or {}
    build = det.get("build") or {}
    variant = det.get("kernel_variant", "") + ("+packed" if det.get("packed_copy") else "")
    rows.append((os.path.basename(f)[:-5], c["matrix"], c["C"], c["sigma"], d["dtype"],
                 det.get("beta"), variant, det.get("executed_layout"),
                 r["kernel_ms"], d["value"], r["achieved"], r["frac"],
                 det.get("parity_vs_oracle"), d["e2e"]["value"], cpu.get("value"),
                 build.get("device_ms"), (d.get("clocks") or {}).get("sm_mhz"),
                 ",".join((d.get("clocks") or {}).get("reasons") or []) or "-"))
print("# Config sweep (one B200, `sh tools/sweep.sh`)\n")
print("GF/s = 2·nnz/t (padding excluded); GB/s = algorithmic bytes (V_alg) / kernel time; "
      "frac of MEASURED_PEAKS hbm_gbs (measured copy).  parity = device arrays and y "
      "bit-exact vs the oracle (cfg5: 8 blocks of 65,536 rows; None = not checked in that "
      "run).  executed = the layout whole-matrix SpMVs stream (a SELL-32 shadow copy of "
      "the same rows when the build's timed cost model keeps one; `_asbuilt` runs force "
      "the caller's layout, SELLB_SHADOW=0).  ref CPU = the reference's compiled core "
      "(oracle/_ref) on the box's 16 host threads, bounded sample.  build = device build "
      "(CUDA events, shadow included).\n")
print("| run | matrix | C | σ | dtype | β | variant | executed | kernel ms | GF/s | GB/s (alg) "
      "| frac | parity | e2e GF/s | ref CPU GF/s | build ms | SM MHz | throttle |")
print("|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|---|")
for r in rows:
    print("| " + " | ".join(str(v) for v in r) + " |")
