#!/usr/bin/env python3
"""Refresh profiles/r01_sweep.md, profiles/r01_sweep/ and the DESIGN.md
measured table from one tools/sweep.sh run:  python tools/design_table.py gpurun_out/DIR"""
import glob
import json
import os
import shutil
import subprocess
import sys

d0 = sys.argv[1]
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
R = {}
for f in glob.glob(os.path.join(d0, "*.json")):
    try:
        R[os.path.basename(f)[:-5]] = json.loads(open(f).read().strip().splitlines()[-1])
    except (ValueError, IndexError):
        pass
# profiles/r01_sweep.md: replace the table, keep the header text
tbl = subprocess.run([sys.executable, os.path.join(ROOT, "tools", "sweep_table.py"), d0],
                     capture_output=True, text=True).stdout.split("\n")
sp = os.path.join(ROOT, "profiles", "r01_sweep.md")
old = open(sp).read().split("\n")
j = next(k for k, l in enumerate(old) if l.startswith("| run"))
k = j
while k < len(old) and old[k].startswith("|"):
    k += 1
i = next(k for k, l in enumerate(tbl) if l.startswith("| run"))
m = i
while m < len(tbl) and tbl[m].startswith("|"):
    m += 1
open(sp, "w").write("\n".join(old[:j] + tbl[i:m] + old[k:]))
sd = os.path.join(ROOT, "profiles", "r01_sweep")
shutil.rmtree(sd, ignore_errors=True)
os.makedirs(sd)
for f in glob.glob(os.path.join(d0, "*.json")):
    shutil.copy(f, sd)


def one(key, label, layout, beta, parity, bold=False):
    d = R[key]
    r = d["roofline"]
    c = d.get("cpu_baseline") or {}
    cv = f"{c['value']:.1f}" if c.get("value") else "—"
    v = f"**{d['value']:.0f}**" if bold else f"{d['value']:.0f}"
    return (f"| {label} | {layout} | {beta} | {r['kernel_ms'] * 1e3:.1f} | {v} | "
            f"{r['achieved']:.0f} | {r['frac']:.3f} | {parity} | {cv} | {d['e2e']['value']:.0f} |")


def span(keys, label, layout, beta):
    ds = [R[k] for k in keys]

    def mm(xs, f):
        return f"{f(min(xs))}–{f(max(xs))}"
    return (f"| {label} | {layout} | {beta} | "
            f"{mm([d['roofline']['kernel_ms'] * 1e3 for d in ds], lambda v: f'{v:.1f}')} | "
            f"{mm([d['value'] for d in ds], lambda v: f'{v:.0f}')} | "
            f"{mm([d['roofline']['achieved'] / 1e3 for d in ds], lambda v: f'{v:.1f}')} k | "
            f"{mm([d['roofline']['frac'] for d in ds], lambda v: f'{v:.2f}')} | bit-exact | — | "
            f"{mm([d['e2e']['value'] for d in ds], lambda v: f'{v:.0f}')} |")


Cs = (8, 16, 32, 64, 128)
rows = [
    one("cfg2", "**cfg2 27-pt 128³ (headline)**", "SELL-32-1", "0.9948", "bit-exact", True),
    one("cfg2_f32", "cfg2 fp32", "SELL-32-1", "0.9948", "bit-exact (binary32 oracle)"),
    one("cfg1", "cfg1 5-pt 1000² (L2 flushed)", "SELL-32-1", "0.9996", "bit-exact"),
    one("cfg3_s1", "cfg3 power-law 4M, σ=1", "SELL-32-1", "0.195", "bit-exact"),
    one("cfg3_s128", "cfg3, σ=128", "SELL-32-128", "0.321", "bit-exact"),
    one("cfg3_s512", "cfg3, σ=512", "SELL-32-512", "0.486", "bit-exact"),
    one("cfg3_s4000000", "cfg3, σ=N", "SELL-32-N", "0.999", "bit-exact"),
    span([f"cfg4_C{c}_s2097152" for c in Cs], "cfg4 skewed 2²¹, C=8..128, σ=N", "SELL-C-N", "1.0"),
    span([f"cfg4_C{c}_s1" for c in Cs], "cfg4, C=8..128, σ=1", "SELL-C-1", "0.07–0.56"),
    span([f"cfg4_C{c}_s{16 * c}" for c in Cs], "cfg4, C=8..128, σ=16C", "SELL-C-16C", "0.07–0.56"),
    span([f"cfg4_C{c}_s{16 * c}_f32" for c in Cs], "cfg4 fp32, C=8..128, σ=16C", "SELL-C-16C",
         "0.07–0.56"),
    one("cfg5_s512", "cfg5 banded-random 2²⁶, 1.32e9 nnz", "SELL-32-512", "0.983",
        "bit-exact (3 blocks)", True),
]
dp = os.path.join(ROOT, "DESIGN.md")
s = open(dp).read()
a = s.index("| **cfg2 27-pt 128³ (headline)**")
b = s.index("β is the format occupancy;")
open(dp, "w").write(s[:a] + "\n".join(rows) + "\n\n" + s[b:])
print("\n".join(rows))
