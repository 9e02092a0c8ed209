#!/usr/bin/env python3
"""Benchmark: fp64 SELL-32-sigma SpMV on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--config cfg5|cfg1|cfg2|cfg3|cfg4] [--sigma S] [--dtype f64|f32]

One "step" = one SpMV y = A x over the whole matrix (all chunks), x and the
matrix resident in HBM.  Default workload: BASELINE configs[4] -- the metric
is quoted "at 1/2/4/8 B200" on it -- the N = 2^26 banded-random
Hamiltonian-like matrix (1,321,641,891 nonzeros), SELL-32-512, fp64,
generated and built on the GPU (16 GB of CRS never touches the host).  Its
algorithmic bytes (17 GB) exceed the 126 MB L2 many times over, so no flush
is needed between steps.

N > 1 (``--gpus N``; re-launched under torch.distributed.run when not
already under it; one process per GPU, NCCL): strong scaling of the same
matrix -- N row blocks aligned to lcm(32, 512), each generated and built on
its own GPU, the x halo exchanged over NCCL and overlapped with the interior
chunks (paper_1307_6209_b200/dist.py).  ``--config cfg2`` under N > 1 is the
weak-scaling stencil (one 128^3 z-slab per GPU).

Printed JSON (rank 0): metric/value (GF/s = 2 nnz / t, padding excluded,
bench.py:89 of the reference), roofline of the SpMV kernel against
MEASURED_PEAKS.json hbm_gbs, e2e through the public API the reference's
callers use (``spmv_sell(m, x, y)`` with ordinary pageable NumPy vectors;
the pinned-buffer number beside it), the reference CPU path timed on this
host (cpu_baseline), clocks sampled during the timed region, gpu_launches.

``--impl reference`` times the reference's own compiled kernel core
(oracle/_ref, built from /root/reference sources) with all host threads,
using the reference's static schedule (spmv.py:53-58) on the same layout
(cfg5: a 2^20-row block of the same matrix; the config dict is identical
to our arm's, the block is named in cpu_baseline.sample).
"""

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

REPO = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REPO)

METRIC = "spMVM GFLOP/s (2\u00b7nnz/t) and HBM GB/s vs roofline, fp64, at 1/2/4/8 B200"
UNIT = "GFLOP/s"


def log(*a):
    print(*a, file=sys.stderr, flush=True)


def measured_peaks():
    p = os.path.join(REPO, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# workloads
# ---------------------------------------------------------------------------

def make_matrix(config, rank=0, world=1):
    from paper_1307_6209_b200 import generate
    if config == "cfg1":
        return generate.laplace2d(1000), "2D 5-point Laplacian 1000x1000"
    if config == "cfg2":
        if world == 1:
            return generate.stencil27(128), "3D 27-point stencil 128^3"
        return None, f"3D 27-point stencil 128x128x{128 * world} (z-slabs)"
    if config == "cfg3":
        return generate.powerlaw(4_000_000), "power-law rows N=4M mean~20"
    if config == "cfg4":
        from paper_1307_6209_b200 import coo_to_crs, gen_skewed
        return (coo_to_crs(gen_skewed(1 << 21, 8, 2048, 1024)),
                "skewed N=2^21 base 8, 1024 spikes of 2048 (sellkit gen_skewed)")
    raise SystemExit(f"unknown config {config}")


# ---------------------------------------------------------------------------
# clocks during the timed region
# ---------------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "50"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except OSError:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"],
                    "samples": 0}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except subprocess.TimeoutExpired:
            self.proc.kill()
        self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ("hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap")
        for ln in self.lines:
            f = [t.strip() for t in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


# ---------------------------------------------------------------------------
# CPU baseline: the reference's compiled core (oracle/_ref) on host cores
# ---------------------------------------------------------------------------

def cpu_reference_run(o, x, budget_s=10.0, threads=None, n_chunks=None):
    """Time the reference kernel (oracle/_ref, else the C port) with the
    reference's static chunk split over `threads` host threads.  Returns
    (gflops, kind, cores, sample, seconds_per_rep)."""
    import oracle
    from concurrent.futures import ThreadPoolExecutor
    ref = oracle.ref_kernels()
    kind = "reference" if ref is not None else "port"
    fn = ref.spmv_sell_range if ref is not None else oracle.spmv_sell_range
    threads = threads or os.cpu_count() or 1
    nch = o.n_chunks if n_chunks is None else min(n_chunks, o.n_chunks)
    nnz = int(o.row_lengths[: nch * o.C].sum(dtype=np.int64))
    y = np.zeros(o.n_rows_padded)
    b = np.linspace(0, nch, threads + 1).astype(int)
    spans = [(int(b[t]), int(b[t + 1])) for t in range(threads) if b[t + 1] > b[t]]
    pool = ThreadPoolExecutor(max_workers=len(spans))

    def one():
        list(pool.map(lambda s: fn(o.cs, o.cl, o.C, o.col, o.val, x, y, s[0], s[1], False),
                      spans))
    t0 = time.perf_counter()
    one()                                   # warm-up, also calibrates
    t1 = max(time.perf_counter() - t0, 1e-6)
    reps = max(1, min(1000, int(budget_s / 3 / t1)))
    times = []
    for _ in range(3):
        t0 = time.perf_counter()
        for _ in range(reps):
            one()
        times.append((time.perf_counter() - t0) / reps)
    pool.shutdown()
    best = min(times)
    sample = (f"{nch} of {o.n_chunks} chunks ({nnz} nnz), {reps} reps x 3 trials, best trial; "
              f"static split over {len(spans)} threads (sellkit spmv.py:53-58), "
              f"{'oracle/_ref = reference _kernels.pyx compiled -O3' if ref else 'C port'}")
    return 2.0 * nnz / best / 1e9, kind, len(spans), sample, best


def host_cpu_desc():
    """CPU model, logical CPUs and last-level cache from lscpu."""
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True).stdout
    except OSError:
        return "unknown"
    kv = {}
    for line in out.splitlines():
        if ":" in line:
            k, v = line.split(":", 1)
            kv[k.strip()] = v.strip()
    desc = kv.get("Model name", "unknown")
    if kv.get("CPU(s)"):
        desc += f", {kv['CPU(s)']} logical CPUs"
    if kv.get("L3 cache"):
        desc += f", L3 {kv['L3 cache']}"
    return desc


# ---------------------------------------------------------------------------
# the config dict both arms print (identical, so the driver can compare)
# ---------------------------------------------------------------------------

CFG5_NNZ = {1 << 26: 1_321_641_891}     # generate.hamiltonian_rows, default keep/seed


def workload_desc(args, world):
    if args.config == "cfg5":
        n = args.n or (1 << 26)
        return (f"banded-random Hamiltonian-like N={n} (BASELINE configs[4]), "
                f"SELL-{args.C}-{args.sigma}")
    if args.config == "cfg2" and world > 1:
        return (f"3D 27-point stencil 128x128x{128 * world} in {world} z-slabs "
                f"(weak scaling), SELL-{args.C}-{args.sigma}")
    names = {"cfg1": "2D 5-point Laplacian 1000x1000 (BASELINE configs[0])",
             "cfg2": "3D 27-point stencil 128^3 (BASELINE configs[1])",
             "cfg3": "power-law rows N=4M mean~20 (BASELINE configs[2])",
             "cfg4": "skewed N=2^21 base 8, 1024 spikes of 2048 (BASELINE configs[3])"}
    if args.config not in names:
        raise SystemExit(f"unknown config {args.config}")
    return f"{names[args.config]}, SELL-{args.C}-{args.sigma}"


def bench_config(args, world):
    """Workload identity only; measurement details go under "details"."""
    n_rows = {"cfg1": 1_000_000, "cfg2": 128 ** 3 * max(1, world if args.config == "cfg2"
                                                        else 1),
              "cfg3": 4_000_000, "cfg4": 1 << 21}.get(args.config, args.n or (1 << 26))
    l2 = ("flushed between steps (4xL2 scratch write + half read back); value from the "
          "SpMV's own events") if args.config == "cfg1" else "inputs larger than L2"
    return {"workload": workload_desc(args, world), "matrix": args.config, "C": args.C,
            "sigma": args.sigma, "dtype": args.dtype, "n_rows": n_rows,
            "parallelism": "1 GPU" if world == 1 else f"row-blocks x{world}, NCCL halo",
            "l2": l2}


# ---------------------------------------------------------------------------
# reference arm
# ---------------------------------------------------------------------------

def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    import oracle
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    sigma = args.sigma
    if args.config == "cfg2" and world > 1:
        from paper_1307_6209_b200 import generate
        crs = generate.stencil27(128, nz=128 * world)
        block = f"the whole 128x128x{128 * world} stencil"
    elif args.config == "cfg5":
        # the host cannot hold 1.3e9 nonzeros through the reference's path:
        # a 2^20-row block of the row-addressable matrix
        from paper_1307_6209_b200 import CRSMatrix, generate
        n = args.n or (1 << 26)
        rows = min(n, 1 << 20)
        rp, cl_, vl = generate.hamiltonian_rows(n, 0, rows)
        crs = CRSMatrix(rows, n, rp, cl_, vl)
        block = f"rows [0, {rows}) of the N={n} matrix (the full matrix is 16 GB of CRS)"
    else:
        crs, _ = make_matrix(args.config)
        block = "the whole matrix"
    o = oracle.crs_to_sell(crs.rpt, crs.col, crs.val, crs.n_rows, crs.n_cols, args.C, sigma)
    x = np.random.default_rng(12345).uniform(-1, 1, crs.n_cols)
    threads = os.cpu_count() or 1
    # size each step so warmup + steps finish within ~2 minutes
    gf_probe, kind, cores, _, t_full = cpu_reference_run(o, x, budget_s=1.0, threads=threads)
    total_steps = args.steps + args.warmup
    frac = min(1.0, 120.0 / max(total_steps * t_full, 1e-9))
    nch = max(1, int(o.n_chunks * frac))
    ref = oracle.ref_kernels()
    fn = ref.spmv_sell_range if ref is not None else oracle.spmv_sell_range
    from concurrent.futures import ThreadPoolExecutor
    b = np.linspace(0, nch, threads + 1).astype(int)
    spans = [(int(b[t]), int(b[t + 1])) for t in range(threads) if b[t + 1] > b[t]]
    y = np.zeros(o.n_rows_padded)
    nnz = int(o.row_lengths[: nch * o.C].sum(dtype=np.int64))
    with ThreadPoolExecutor(max_workers=len(spans)) as pool:
        def step():
            list(pool.map(lambda s: fn(o.cs, o.cl, o.C, o.col, o.val, x, y, s[0], s[1],
                                       False), spans))
        for _ in range(args.warmup):
            step()
        t0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        dt = time.perf_counter() - t0
    value = 2.0 * nnz * args.steps / dt / 1e9
    sample = (f"{block}: {nch} of {o.n_chunks} chunks ({nnz} nnz) per step; static split "
              f"over {len(spans)} threads (sellkit spmv.py:53-58); "
              f"{'reference _kernels.pyx compiled from /root/reference sources (oracle/_ref)' if ref else 'C port (oracle/sell_oracle.c)'}; "
              f"host {host_cpu_desc()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 4), "unit": UNIT,
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(dt / args.steps * 1e3, 4), "higher_is_better": True,
        "scaling": "strong" if args.config == "cfg5" and world > 1 else "weak",
        "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": bench_config(args, world),
        "cpu_baseline": {"value": round(value, 4), "unit": UNIT, "cores": len(spans),
                         "kind": "reference" if ref is not None else "port",
                         "sample": sample},
        "e2e": {"value": round(value, 4), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our arm
# ---------------------------------------------------------------------------

def model_block(s, nnz, n_rows, n_cols, n_pad, n_chunks, slots, s_v, traffic, kern_ms, peak):
    """The paper's performance model next to the measurement (model.py):
    beta, sector beta_eff, code balance with ideal alpha and the predicted
    P = b/B, and -- when an ncu capture of this layout is committed -- the
    measured balance and alpha from DRAM bytes."""
    from paper_1307_6209_b200 import model
    out = {"beta": round(nnz / slots, 6) if slots else 1.0}
    try:
        be, vs, cs_ = s.sector_occupancy()
        out["beta_eff"] = round(be, 6)
    except Exception:                      # imported without row lengths
        vs = cs_ = None
    if nnz and n_rows and n_cols and slots:
        nzr, nzc = nnz / n_rows, nnz / n_cols
        if s_v == 8:
            bal = model.code_balance_sell(1.0 / nzc, nnz / slots, nzr)
            out["B_paper_ideal_alpha"] = round(bal, 4)
            out["P_paper_GFs"] = round(peak / bal, 1)
        out["B_alg"] = round(model.algorithmic_bytes(nnz, n_cols, n_pad, n_chunks, s_v=s_v)
                             / (2.0 * nnz), 4)
        if traffic and s_v == 8:
            out["B_measured"] = round(traffic / (2.0 * nnz), 4)
            a = model.infer_alpha(traffic, nnz, nnz / slots, nzr, line_bytes=32)
            out["alpha_paper"] = round(a.alpha, 4)
            out["alpha_ideal"] = round(1.0 / nzc, 4)
            try:                           # bytes the kernels stream as configured
                mat, _, extra = s.streamed_bytes()
            except Exception:
                mat = None
            if mat is not None:
                out["alpha_eff"] = round(model.alpha_from_traffic(
                    traffic, nnz, mat, n_pad, n_chunks, extra_bytes=extra).alpha, 4)
            out["traffic_source"] = "profiles/ncu_traffic.json (ncu dram bytes, one launch)"
        if s_v == 8 and nnz <= 200_000_000 and hasattr(s, "handle"):
            # the reference's LRU model (cachesim.py:49-75) with an L2-sized
            # fully-associative cache of 32 B lines, replayed on the device
            try:
                import torch
                from paper_1307_6209_b200 import cachesim
                l2 = (torch.cuda.get_device_properties(0).L2_cache_size // 32) * 32
                v_sim = cachesim.simulate_rhs_traffic(s, l2, 32)
                out["alpha_sim_lru_l2"] = round(
                    model.infer_alpha(v_sim, nnz, nnz / slots, nzr, line_bytes=32).alpha, 4)
            except Exception as e:         # reported, never fatal for the bench line
                out["alpha_sim_lru_l2"] = f"unavailable: {type(e).__name__}"
    return out


def load_profile_traffic(key):
    p = os.path.join(REPO, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    with open(p) as f:
        d = json.load(f)
    v = d.get(key)
    return None if v is None else float(v)


ARRAYS = ("cs", "cl", "col", "val", "perm", "row_lengths")


def host_workload(args, dt_np):
    """cfg1-cfg4: CRS generated on the host, built on the GPU."""
    import torch
    import oracle
    import paper_1307_6209_b200 as sb
    crs, desc = make_matrix(args.config)
    x = np.random.default_rng(12345).uniform(-1, 1, crs.n_cols).astype(dt_np)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    s = sb.crs_to_sell(crs, args.C, args.sigma, dtype=dt_np)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    # the device build alone (CRS already in HBM), timed with CUDA events
    dev = torch.device("cuda", 0)
    rpt_d = torch.from_numpy(crs.rpt).to(dev)
    col_d = torch.from_numpy(crs.col).to(dev)
    val_d = torch.from_numpy(crs.val.astype(dt_np)).to(dev)
    sb.crs_to_sell_device(rpt_d, col_d, val_d, crs.n_rows, crs.n_cols, args.C, args.sigma).free()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s2 = sb.crs_to_sell_device(rpt_d, col_d, val_d, crs.n_rows, crs.n_cols, args.C, args.sigma)
    e1.record()
    e1.synchronize()
    s2.free()                       # after the closing event (cudaFree is synchronous)
    build_dev_ms = e0.elapsed_time(e1)
    del rpt_d, col_d, val_d
    t0 = time.perf_counter()
    oracle.crs_to_sell(crs.rpt, crs.col, crs.val, crs.n_rows, crs.n_cols, args.C, args.sigma)
    build_cpu_s = time.perf_counter() - t0

    def parity(yd):
        o = oracle.crs_to_sell(crs.rpt, crs.col, crs.val.astype(dt_np), crs.n_rows,
                               crs.n_cols, args.C, args.sigma)
        y_ref = oracle.spmv_sell(o, x, threads=os.cpu_count() or 1)
        ok = yd.cpu().numpy().tobytes() == y_ref.tobytes()
        return ok and all(getattr(s, k).tobytes() == getattr(o, k).tobytes() for k in ARRAYS)

    def cpu(budget):
        o = oracle.crs_to_sell(crs.rpt, crs.col, crs.val, crs.n_rows, crs.n_cols, 32,
                               args.sigma)
        gf, kind, cores, sample, _ = cpu_reference_run(o, x.astype(np.float64),
                                                       budget_s=budget)
        # the same kernel on one thread (T = 1 and T = all)
        gf1, _, _, _, _ = cpu_reference_run(o, x.astype(np.float64),
                                            budget_s=min(4.0, budget / 3), threads=1)
        return {"value": round(gf, 4), "unit": UNIT, "cores": cores, "kind": kind,
                "value_1thread": round(gf1, 4),
                "sample": sample + f"; host {host_cpu_desc()}"}

    b = build_roofline(s.info(), dt_np, build_dev_ms, build_s,
                       note="device_ms: crs_to_sell on CRS already in HBM (CUDA events); "
                            "host_s adds the pageable H2D of the CRS; cpu: the C "
                            "restatement of formats.py:295-393 (oracle), one thread")
    b["cpu_port_1thread_s"] = round(build_cpu_s, 4)
    return {"sell": s, "desc": desc, "x": x, "build_s": build_s, "parity": parity, "cpu": cpu,
            "build": b}


def build_roofline(info, dt_np, device_ms, host_s, note=""):
    """Bytes the device build (crs_to_sell, formats.py:295-393) must move at
    least -- read the CRS, write the SELL arrays (cs, cl, col, val,
    row_lengths, perm, order) -- against its CUDA-event time."""
    s_v = 4 if dt_np == np.float32 else 8
    n, n_pad, nch = info.n_rows, info.n_rows_padded, info.n_chunks
    nnz, slots = info.nnz, info.slots
    read = 8 * (n + 1) + (4 + s_v) * nnz
    write = 12 * nch + 8 + (4 + s_v) * slots + 4 * n_pad + 4 * n + 4 * n_pad
    gbs = (read + write) / (device_ms / 1e3) / 1e9 if device_ms > 0 else None
    peak, _ = measured_peaks()
    return {"device_ms": round(device_ms, 3), "host_s": round(host_s, 4),
            "includes": "sort, layout, fill, variant cost model" + (
                ", the SELL-32 shadow copy (DESIGN.md 4.2)" if info.shadow else ""),
            "bytes_alg": int(read + write),
            "achieved_gbs": round(gbs, 1) if gbs else None,
            "frac_of_hbm": round(gbs / peak, 4) if gbs else None, "note": note}


def parity_blocks(n, blk):
    """Row blocks checked against the oracle at full size: the first, the
    last, and blocks straddling each quarter boundary (the N = 2/4 rank
    boundaries of the row-partitioned run), aligned to the block size."""
    starts = {0, max(0, n - blk)}
    for q in (1, 2, 3):
        b = (n * q // 4) // blk * blk
        starts.add(max(0, min(n - blk, b - blk // 2)))   # straddles b (512-aligned)
        starts.add(max(0, min(n - blk, b)))
    return sorted(starts)


def cfg5_workload(args, dt_np):
    """cfg5: the N = 2^26, ~1.3e9-nonzero banded-random matrix generated and
    built on the GPU (16 GB of CRS never touches the host).  Parity and the
    CPU baseline use row blocks regenerated on the host (row-addressable
    generator; block builds equal slices of the global build)."""
    import torch
    import oracle
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import CRSMatrix, generate
    n = args.n or (1 << 26)
    sigma = args.sigma
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rpt, col, val = generate.hamiltonian_device(n, device=0, dtype=dt_np)
    torch.cuda.synchronize()
    t_gen = time.perf_counter() - t0
    s = sb.crs_to_sell_device(rpt, col, val, n, n, args.C, sigma)
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0 - t_gen
    # the device build alone, timed with CUDA events (a second build of the
    # same CRS; the build returns once its stream is idle, and the matrix is
    # freed after the closing event)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    s2 = sb.crs_to_sell_device(rpt, col, val, n, n, args.C, sigma)
    e1.record()
    e1.synchronize()
    s2.free()
    build_dev_ms = e0.elapsed_time(e1)
    del rpt, col, val
    torch.cuda.empty_cache()
    x = np.random.default_rng(12345).uniform(-1, 1, n).astype(dt_np)
    blk = 1 << 16

    def block(r0, r1):
        rp, cl_, vl = generate.hamiltonian_rows(n, r0, r1)
        return CRSMatrix(r1 - r0, n, rp, cl_, vl.astype(dt_np) if dt_np == np.float32 else vl)

    def parity(yd):
        ok = True
        for r0 in parity_blocks(n, blk):
            b = block(r0, r0 + blk)
            o = oracle.crs_to_sell(b.rpt, b.col, b.val, b.n_rows, n, args.C, sigma)
            got = s.export_range(r0 // 32, (r0 + blk) // 32)
            for k in ("cs", "cl", "col", "val", "row_lengths"):
                ok = ok and got[k].tobytes() == getattr(o, k).tobytes()
            y_ref = oracle.spmv_sell(o, x)
            ok = ok and yd[r0:r0 + blk].cpu().numpy().tobytes() == y_ref.tobytes()
        return ok

    def cpu(budget):
        b = block(0, min(n, 1 << 20))
        o = oracle.crs_to_sell(b.rpt, b.col, b.val.astype(np.float64), b.n_rows, n, args.C, sigma)
        gf, kind, cores, sample, _ = cpu_reference_run(o, x.astype(np.float64),
                                                       budget_s=budget)
        return {"value": round(gf, 4), "unit": UNIT, "cores": cores, "kind": kind,
                "sample": f"rows [0, {b.n_rows}) block of the N={n} matrix: " + sample
                          + f"; host {host_cpu_desc()}"}

    scope = (f"{len(parity_blocks(n, blk))} blocks of {blk} rows (first, last, quarter "
             f"boundaries): cs/cl/col/val/row_lengths and y bit-exact vs the oracle")
    info = s.info()
    return {"sell": s, "parity_scope": scope,
            "build": build_roofline(info, dt_np, build_dev_ms, build_s,
                                    note="device_ms: crs_to_sell_device on the device-"
                                         "generated CRS (CUDA events); generation "
                                         f"{t_gen:.3f} s"),
            "desc": f"banded-random Hamiltonian-like N={n} (device-generated, "
                               f"generation {t_gen:.2f} s)",
            "x": x, "build_s": build_s, "parity": parity, "cpu": cpu}


def run_ours(args):
    import torch
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world > 1 or os.environ.get("SELLB_FORCE_DIST"):   # (1-rank smoke of the N>1 leg)
        import bench_dist
        args.peak = measured_peaks()[0]
        args.metric = METRIC
        args.config_dict = bench_config(args, world)
        args.clock_sampler = ClockSampler
        return bench_dist.bench_main(args)
    import oracle
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import _lib
    from paper_1307_6209_b200.model import algorithmic_bytes

    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    dt_np = np.float32 if args.dtype == "f32" else np.float64
    tdt = torch.float32 if args.dtype == "f32" else torch.float64
    sigma = args.sigma
    wl = (cfg5_workload if args.config == "cfg5" else host_workload)(args, dt_np)
    s, desc, x_host, build_s = wl["sell"], wl["desc"], wl["x"], wl["build_s"]
    info = s.info()
    n_rows, n_cols = info.n_rows, info.n_cols
    nnz, n_pad, n_chunks, slots = info.nnz, info.n_rows_padded, info.n_chunks, info.slots
    s_v = 4 if args.dtype == "f32" else 8
    v_alg = algorithmic_bytes(nnz, n_cols, n_pad, n_chunks, s_v=s_v)
    lib = _lib.load()
    handle = s.handle

    xd = torch.from_numpy(x_host).to(dev)
    yd = torch.zeros(n_pad, dtype=tdt, device=dev)
    stream = torch.cuda.current_stream(dev)
    sp = stream.cuda_stream

    def launch():
        _lib.check(lib.sellb_spmv(handle, xd.data_ptr(), yd.data_ptr(), 0, n_chunks, 0,
                                  0, sp))

    # parity gate on the benchmarked matrix (oracle is the checker only)
    launch()
    torch.cuda.synchronize()
    parity = None
    if not args.skip_parity:
        parity = bool(wl["parity"](yd))
        if not parity:
            log("PARITY FAILURE against the oracle")

    for _ in range(args.warmup):
        launch()
    torch.cuda.synchronize()

    # inputs smaller than ~2x L2 are flushed between steps (timing hygiene)
    l2_bytes = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = None
    if v_alg < 2 * l2_bytes:
        flush = torch.empty(4 * l2_bytes, dtype=torch.uint8, device=dev)

    # timed region: K steps, per-step events on the launching stream
    # Without a flush every step is exactly one SpMV launch, back to back on
    # one stream, so the region's two events give the average launch time
    # (per-launch event pairs would add ~3 us of gap per launch).  With a
    # flush, each SpMV gets its own event pair and the flushes are excluded.
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(args.steps)] if flush is not None else []
    clocks = ClockSampler(0)
    clocks.start()
    time.sleep(0.25)
    for _ in range(3):                 # re-warm after the idle sampler start
        launch()
    torch.cuda.synchronize()
    t_start = torch.cuda.Event(enable_timing=True)
    t_end = torch.cuda.Event(enable_timing=True)
    n_launch0 = lib.sellb_launch_count()     # the library counts every kernel it launches
    t_start.record(stream)
    for i in range(args.steps):
        if flush is not None:           # outside the kernel's event pair
            _lib.check(lib.sellb_l2_flush(flush.data_ptr(), flush.numel(), sp))
            ev[i][0].record(stream)
            launch()
            ev[i][1].record(stream)
        else:
            launch()
    t_end.record(stream)
    n_launches = lib.sellb_launch_count() - n_launch0
    torch.cuda.synchronize()
    clk = clocks.stop()
    total_ms = t_start.elapsed_time(t_end)
    if flush is not None:
        kern_ms = statistics.mean(a.elapsed_time(b) for a, b in ev)
    else:
        kern_ms = total_ms / args.steps
    # with an L2 flush between steps the step time is the SpMV's own events
    step_ms = kern_ms if flush is not None else total_ms / args.steps
    value = 2.0 * nnz / (step_ms / 1e3) / 1e9
    peak, peak_kind = measured_peaks()
    achieved = v_alg / (kern_ms / 1e3) / 1e9

    # e2e through the public API a reference caller uses: spmv_sell(m, x, y)
    # with ordinary (pageable) NumPy vectors (spmv.py:105-122) -- x H2D,
    # the product, y D2H, all inside every timed call
    e2e_steps = max(3, min(args.steps, 100))
    x_np = np.array(x_host, dtype=dt_np)            # plain pageable arrays
    y_np = np.empty(n_pad, dtype=dt_np)
    for _ in range(2):
        sb.spmv_sell(s, x_np, y_np)
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        sb.spmv_sell(s, x_np, y_np)
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    e2e_ok = bool(y_np.tobytes() == yd.cpu().numpy().tobytes())
    # the same call with y=None (the reference allocates y per call)
    t0 = time.perf_counter()
    n_alloc = max(2, min(e2e_steps, 10))
    for _ in range(n_alloc):
        y_new = sb.spmv_sell(s, x_np)
    e2e_alloc_s = (time.perf_counter() - t0) / n_alloc
    del y_new
    # and through the C ABI with library-pinned x / y (PCIe-bound floor)
    import ctypes
    px, py = ctypes.c_void_p(), ctypes.c_void_p()
    _lib.check(lib.sellb_host_alloc(n_cols * s_v, ctypes.byref(px)))
    _lib.check(lib.sellb_host_alloc(n_pad * s_v, ctypes.byref(py)))
    xh = np.ctypeslib.as_array((ctypes.c_byte * (n_cols * s_v)).from_address(px.value)).view(dt_np)
    yh = np.ctypeslib.as_array((ctypes.c_byte * (n_pad * s_v)).from_address(py.value)).view(dt_np)
    xh[:] = x_host
    for _ in range(3):
        _lib.check(lib.sellb_spmv_host(handle, px.value, py.value, 0, n_chunks, 0, 0, sp))
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        _lib.check(lib.sellb_spmv_host(handle, px.value, py.value, 0, n_chunks, 0, 0, sp))
    e2e_pin_s = (time.perf_counter() - t0) / e2e_steps
    e2e_ok = e2e_ok and bool(yh.tobytes() == y_np.tobytes())
    lib.sellb_host_free(px)
    lib.sellb_host_free(py)
    del x_np, y_np

    # reference CPU path on this host, bounded sample (rank 0, N=1)
    cpu = None
    if not args.skip_cpu:
        cpu = wl["cpu"](args.cpu_budget)

    shadow = bool(getattr(s, "shadow", False))
    traffic = load_profile_traffic(f"{args.config}_s{sigma}_{args.dtype}"
                                   + ("_shadow" if shadow else "")) if args.C == 32 else None
    line = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": 1,
        "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(step_ms, 5), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
        "config": bench_config(args, 1),
        "details": {"matrix": desc, "n_rows": n_rows, "nnz": nnz, "slots": slots,
                    "beta": round(nnz / slots, 6), "kernel_variant": s.variant,
                    "packed_copy": s.packed,
                    # irregular layouts: whole-matrix SpMVs stream a device-built
                    # SELL-32-N (x in L2) or SELL-32-512 copy of the same rows and
                    # scatter each row's sum back (bit-exact); SELLB_SHADOW=0 times
                    # the layout as built
                    "shadow_layout": shadow,
                    "executed_layout": ("SELL-32-%s shadow of the stored rows, sums "
                                        "scattered to the SELL-%d-%d rows" % (
                                            "N" if s.shadow_sigma >= n_pad else s.shadow_sigma,
                                            args.C, sigma))
                    if shadow else "SELL-%d-%d as built" % (args.C, sigma),
                    "long_rows": s.long_rows_info(),
                    "l2": ("flushed between steps (%d MB scratch write, then half of it "
                           "read back so the L2 holds clean lines); value from the SpMV's "
                           "own events" % (4 * l2_bytes // 2**20)) if flush is not None
                    else "inputs larger than L2 (V_alg %.0f MB > %d MB L2)" % (
                        v_alg / 1e6, l2_bytes // 2**20),
                    "build_s": round(build_s, 4), "build": wl.get("build"),
                    "parity_vs_oracle": parity, "parity_scope": wl.get("parity_scope")},
        "model": model_block(s, nnz, n_rows, n_cols, n_pad, n_chunks, slots, s_v, traffic,
                             kern_ms, peak),
        "roofline": {"bound": "hbm", "achieved": round(achieved, 2), "peak": peak,
                     "unit": "GB/s", "frac": round(achieved / peak, 4),
                     "traffic": traffic, "peak_source": f"{peak_kind} hbm_gbs (copy)",
                     "bytes_alg_per_launch": v_alg,
                     "kernel_ms": round(kern_ms, 5)},
        "e2e": {"value": round(2.0 * nnz / e2e_s / 1e9, 3), "unit": UNIT,
                "h2d_bytes_per_step": n_cols * s_v, "d2h_bytes_per_step": n_pad * s_v,
                "ms_per_step": round(e2e_s * 1e3, 4),
                "api": "paper_1307_6209_b200.spmv_sell(m, x, y) with pageable NumPy x / y "
                       "(the reference's call, spmv.py:105-122)",
                "matches_device": e2e_ok,
                "y_allocated_per_call": {"value": round(2.0 * nnz / e2e_alloc_s / 1e9, 3),
                                         "ms_per_step": round(e2e_alloc_s * 1e3, 4),
                                         "api": "spmv_sell(m, x) (y=None)"},
                "pinned": {"value": round(2.0 * nnz / e2e_pin_s / 1e9, 3),
                           "ms_per_step": round(e2e_pin_s * 1e3, 4),
                           "api": "sellb_spmv_host with library-pinned x / y"}},
        "cpu_baseline": cpu,
        "clocks": clk,
        "gpu_launches": int(n_launches),
    }
    print(json.dumps(line), flush=True)
    return 0


def free_port():
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        return so.getsockname()[1]


def relaunch_distributed(args, argv):
    """`bench.py --gpus N` outside torchrun: re-exec under
    torch.distributed.run, one process per GPU (the driver's own launch)."""
    import torch
    have = torch.cuda.device_count()
    if have < args.gpus:
        raise SystemExit(f"--gpus {args.gpus} asks for {args.gpus} GPUs, {have} visible")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={free_port()}", os.path.abspath(__file__)] + list(argv)
    log("relaunching:", " ".join(cmd))
    os.execv(sys.executable, cmd)


def main(argv=None):
    argv = sys.argv[1:] if argv is None else argv
    ap = argparse.ArgumentParser(description=__doc__.splitlines()[0])
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--impl", choices=("ours", "reference"), default="ours")
    ap.add_argument("--config", default="cfg5",
                    choices=("cfg1", "cfg2", "cfg3", "cfg4", "cfg5"))
    ap.add_argument("--sigma", type=int, default=None,
                    help="sorting scope (default 512 for cfg5, else 1)")
    ap.add_argument("--C", type=int, default=32, help="chunk height")
    ap.add_argument("--dtype", choices=("f64", "f32"), default="f64")
    ap.add_argument("--skip-parity", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--cpu-budget", type=float, default=12.0)
    # --rows: under torchrun a bare --n is an ambiguous prefix of its own options
    ap.add_argument("--n", "--rows", dest="n", type=int, default=0,
                    help="cfg5 rows (default 2^26)")
    args = ap.parse_args(argv)
    if args.sigma is None:
        args.sigma = 512 if args.config == "cfg5" else 1
    if args.warmup < 3:
        args.warmup = 3
    world = os.environ.get("WORLD_SIZE")
    if world is not None and int(world) != args.gpus and args.gpus != 1:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if world is not None:
        args.gpus = int(world)
    if args.impl == "reference":
        return run_reference(args)
    if world is None and args.gpus > 1:
        relaunch_distributed(args, argv)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
