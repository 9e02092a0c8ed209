#!/usr/bin/env python3
"""Condense an ncu report (or a launch-list CSV) into the summary committed
under profiles/.

    python tools/ncu_summary.py rep  gpurun_out/prof.ncu-rep  [bytes_alg]
    python tools/ncu_summary.py list gpurun_out/launches.csv
"""
import csv
import io
import subprocess
import sys
from collections import OrderedDict

SECTIONS = ("GPU Speed Of Light Throughput", "Memory Workload Analysis", "Occupancy",
            "Launch Statistics", "Warp State Statistics")
RAW = ("gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
       "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
       "sm__warps_active.avg.pct_of_peak_sustained_active",
       "launch__registers_per_thread", "lts__t_sector_hit_rate.pct",
       "smsp__average_warp_latency_issue_stalled_long_scoreboard",
       "l1tex__t_sector_hit_rate.pct")


def rep(path, bytes_alg=None):
    det = subprocess.run(["ncu", "-i", path, "--page", "details", "--csv"],
                         capture_output=True, text=True).stdout
    rows = list(csv.DictReader(io.StringIO(det)))
    by_id = OrderedDict()
    for r in rows:
        by_id.setdefault(r["ID"], []).append(r)
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    rr = list(csv.reader(io.StringIO(raw)))
    hdr, units = rr[0], rr[1]
    for i, (kid, rs) in enumerate(by_id.items()):
        print(f"== launch {kid}: {rs[0]['Kernel Name'][:110]}")
        print(f"   block {rs[0]['Block Size']} grid {rs[0]['Grid Size']}")
        for r in rs:
            if r["Section Name"] in SECTIONS and r["Metric Name"]:
                print(f"   [{r['Section Name'][:18]:18}] {r['Metric Name']:45} "
                      f"{r['Metric Value']:>14} {r['Metric Unit']}")
        if i + 2 < len(rr):
            d = dict(zip(hdr, rr[i + 2]))
            for k in RAW:
                if k in d:
                    print(f"   [raw] {k:60} {d[k]} {units[hdr.index(k)]}")
            if bytes_alg:
                try:
                    rd = float(d["dram__bytes_read.sum"])
                    wr = float(d["dram__bytes_write.sum"])
                    ur = units[hdr.index("dram__bytes_read.sum")]
                    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[ur]
                    uw = units[hdr.index("dram__bytes_write.sum")]
                    scw = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}[uw]
                    t = (rd * scale + wr * scw)
                    print(f"   traffic (read+write) = {t:.0f} B; algorithmic = {bytes_alg} B; "
                          f"ratio = {t / float(bytes_alg):.4f}")
                except (KeyError, ValueError):
                    pass


def launches(path):
    lines = open(path).read().splitlines()
    start = next(i for i, l in enumerate(lines) if l.startswith('"ID"'))
    rows = list(csv.DictReader(io.StringIO("\n".join(lines[start:]))))
    agg = OrderedDict()
    total = 0.0
    for r in rows:
        if r.get("Metric Name") != "gpu__time_duration.sum":
            continue
        v = float(r["Metric Value"]) * {"ns": 1e-3, "us": 1, "usecond": 1, "ms": 1e3,
                                        "nsecond": 1e-3, "msecond": 1e3}.get(r["Metric Unit"], 1)
        name = r["Kernel Name"].split("(")[0][:80]
        n, s = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, s + v)
        total += v
    print(f"{'kernel':80} {'launches':>8} {'total us':>10} {'avg us':>9} {'share':>6}")
    for k, (n, s) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        print(f"{k:80} {n:8d} {s:10.1f} {s / n:9.2f} {s / total:6.1%}")


if __name__ == "__main__":
    if sys.argv[1] == "rep":
        rep(sys.argv[2], sys.argv[3] if len(sys.argv) > 3 else None)
    else:
        launches(sys.argv[2])
