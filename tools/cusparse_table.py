#!/usr/bin/env python3
"""Markdown table of tools/cusparse_compare.py JSON lines:
    python tools/cusparse_table.py profiles/r02_cusparse.jsonl"""
import json
import sys

ARMS = ("ours_sell32_s1", "ours_sell32_sN", "ours_crs", "ours_crs_unrolled",
        "cusparse_csr_alg1", "cusparse_csr_alg2", "cusparse_sell32_alg1")
print("| config | dtype | ours SELL-32-1 | ours SELL-32-N | ours CRS | ours CRS unrolled "
      "| cuSPARSE CSR ALG1 | CSR ALG2 | cuSPARSE SELL-32 |")
print("|---|---|---|---|---|---|---|---|---|")
for line in open(sys.argv[1]):
    if not line.strip():
        continue
    d = json.loads(line)
    cells = []
    for a in ARMS:
        r = d["arms"].get(a)
        cells.append(f"{r['gflops']:.0f} ({r['max_rel_err']:.0e})" if r else "—")
    print(f"| {d['config']} {d['matrix']} | {d['dtype']} | " + " | ".join(cells) + " |")
