#!/usr/bin/env python3
"""Top SASS instructions by warp-stall samples from an ncu report.
    python tools/ncu_hot.py gpurun_out/prof.ncu-rep [N]"""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv"], capture_output=True,
                     text=True).stdout
lines = out.splitlines()
start = next(i for i, l in enumerate(lines) if l.startswith('"Address"'))
rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
tot = sum(float(r["Warp Stall Sampling (All Samples)"] or 0) for r in rows) or 1
rows.sort(key=lambda r: -float(r["Warp Stall Sampling (All Samples)"] or 0))
print(f"total samples {tot:.0f}; {lines[0][:160]}")
for r in rows[:n]:
    s = float(r["Warp Stall Sampling (All Samples)"] or 0)
    print(f"{s / tot:6.1%}  {r['Address'][-5:]}  {r['Source'].strip()[:70]:70}  exec {r['Instructions Executed']}")
