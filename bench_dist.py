"""Multi-GPU leg of bench.py (torchrun, one process per GPU, NCCL).

Lives beside bench.py, outside the product package: it uses the CPU oracle
as the parity checker for each rank's block, which the package never
imports.
"""


import numpy as np
import torch
import torch.distributed as tdist


def time_parts(ds, device, iters):
    """The step's parts alone, eager, CUDA events on the compute stream, max
    over ranks: the halo exchange (post + wait), the interior chunks, the
    boundary chunks; plus the bytes this rank receives per step."""
    st = torch.cuda.current_stream(device)

    def timed(fn):
        tdist.barrier()
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(iters):
            fn()
        e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / iters

    def exchange():
        for w in ds._post_exchange():
            w.wait()

    vals = [timed(exchange),
            timed(lambda: ds.engine.run_ranges(ds.interior, ds.x_full, ds.y)),
            timed(lambda: ds.engine.run_ranges(ds.boundary, ds.x_full, ds.y)),
            float(ds.plan.bytes_per_step(ds.y.element_size()))]
    t = torch.tensor(vals, dtype=torch.float64, device=device)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    ex, it, bd, hb = t.tolist()
    return {"exchange_ms": round(ex, 5), "interior_ms": round(it, 5),
            "boundary_ms": round(bd, 5), "halo_bytes_per_rank_max": int(hb)}


def bench_main(args):
    """Multi-GPU benchmark under torchrun (one process per GPU, NCCL).

    cfg5 (default, BASELINE configs[4]) -- strong scaling: the N = 2^26
    banded-random matrix split into N row blocks, each generated and built on
    its own GPU, halo over the +-65536 / +-2^20 hops.  cfg2 -- weak scaling:
    the 27-point stencil on 128 x 128 x (128 N), one 128^3 z-slab per GPU,
    halo = one 128x128 plane per neighbour."""
    import json
    import os

    import time

    from paper_1307_6209_b200 import generate
    from paper_1307_6209_b200.dist import (_cfg5_bounds, cuda_engine_factory, setup,
                                           setup_device)
    from paper_1307_6209_b200.model import algorithmic_bytes

    # NCCL prints its version banner on fd 1 at communicator creation; the
    # driver reads exactly one JSON line from stdout, so everything but that
    # line goes to stderr
    json_fd = os.dup(1)
    os.dup2(2, 1)
    # communicator lines (ranks, channels, NVLS) on stderr for the record
    os.environ.setdefault("NCCL_DEBUG", "INFO")
    os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    import datetime
    # a wedged peer fails the run within minutes instead of NCCL's default 10
    tdist.init_process_group("nccl", device_id=device,
                             timeout=datetime.timedelta(seconds=300))
    C, sigma = args.C, args.sigma
    dt_np = np.float32 if args.dtype == "f32" else np.float64
    s_v = 4 if args.dtype == "f32" else 8
    if args.config not in ("cfg5", "cfg2"):
        raise SystemExit(f"the row-partitioned leg runs cfg5 (strong) or cfg2 (weak), "
                         f"not {args.config}")
    t0 = time.perf_counter()
    if args.config == "cfg5":
        n_glob = args.n or (1 << 26)
        bounds = _cfg5_bounds(n_glob, world, C, sigma)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        rpt_t, col_t, val_t = generate.hamiltonian_device(n_glob, r0, r1, device=local,
                                                          dtype=dt_np)
        ds = setup_device(rpt_t, col_t, val_t, n_glob, bounds, C, sigma, rank, world, device)
        del rpt_t, col_t, val_t
        torch.cuda.empty_cache()
        scaling = "strong"
        crs = None
    else:
        n, nz_per = 128, 128
        nz = nz_per * world
        n_glob = n * n * nz
        crs = generate.stencil27_slab(n, nz, rank * nz_per, (rank + 1) * nz_per)
        bounds = np.arange(world + 1, dtype=np.int64) * (n * n * nz_per)
        if dt_np == np.float32:
            crs = type(crs)(crs.n_rows, crs.n_cols, crs.rpt, crs.col,
                            crs.val.astype(np.float32))
        ds = setup(crs, bounds, C, sigma, rank, world, device,
                   cuda_engine_factory(C, sigma, device, dtype=dt_np),
                   dtype=torch.float32 if dt_np == np.float32 else torch.float64)
        scaling = "weak"
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    x_glob_rng = np.random.default_rng(12345)
    x_all = x_glob_rng.uniform(-1, 1, n_glob).astype(dt_np)
    ds.x_local.copy_(torch.from_numpy(x_all[ds.r0:ds.r1]))
    sell = ds.engine.sell
    nnz_local = sell.nnz
    n_rows_local = ds.r1 - ds.r0
    # parity of this rank's block against the oracle with the full x --
    # block builds equal slices.  cfg5: the first AND the last
    # 65536 rows of the block, i.e. both halo sides (rows near r0 read the
    # previous rank's x, rows near r1 the next rank's).
    parity = None

    def check_parity():
        import oracle
        ds.step()
        torch.cuda.synchronize()
        y_all = ds.y.cpu().numpy()
        ok = True
        if crs is None:
            from paper_1307_6209_b200.formats import CRSMatrix
            blk = min(1 << 16, n_rows_local)
            for a0 in sorted({0, n_rows_local - blk}):
                rp, cl_, vl = generate.hamiltonian_rows(n_glob, ds.r0 + a0, ds.r0 + a0 + blk)
                chk = CRSMatrix(blk, n_glob, rp, cl_, vl.astype(dt_np))
                o = oracle.crs_to_sell(chk.rpt, chk.col, chk.val, chk.n_rows, chk.n_cols,
                                       C, sigma)
                y_ref = oracle.spmv_sell(o, x_all,
                                         threads=max(1, (os.cpu_count() or 8) // world))
                ok = ok and y_all[a0:a0 + len(y_ref)].tobytes() == y_ref.tobytes()
        else:
            o = oracle.crs_to_sell(crs.rpt, crs.col, crs.val, crs.n_rows, crs.n_cols, C,
                                   sigma)
            y_ref = oracle.spmv_sell(o, x_all, threads=max(1, (os.cpu_count() or 8) // world))
            ok = y_all[:len(y_ref)].tobytes() == y_ref.tobytes()
        return bool(ok)

    if not args.skip_parity:
        parity = check_parity()
    for _ in range(args.warmup):
        ds.step()
    torch.cuda.synchronize()
    # one CUDA graph per step (NCCL post included), opt-in (SELLB_DIST_GRAPH=1):
    # a capture with NCCL traffic between two GPUs has not run yet, and eager
    # posting keeps up with cfg5's per-rank SpMV.  Kept only if its replay
    # from NaN-poisoned halos equals the eager step bitwise on all ranks.
    graphed = False
    if os.environ.get("SELLB_DIST_GRAPH", "0") == "1":
        graphed = ds.capture()
        for _ in range(args.warmup):
            ds.step()
        torch.cuda.synchronize()
        if graphed and not args.skip_parity:      # the replayed step, against the oracle
            parity = bool(parity) and check_parity()
    tdist.barrier()
    st = torch.cuda.current_stream(device)
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    launches0 = ds.engine.lib.sellb_launch_count()
    sampler = args.clock_sampler(local) if rank == 0 else None
    if sampler:
        sampler.start()
        time.sleep(0.25)
    torch.cuda.synchronize()
    tdist.barrier()
    e0.record(st)
    for _ in range(args.steps):
        ds.step()
    e1.record(st)
    torch.cuda.synchronize()
    tdist.barrier()
    clk = sampler.stop() if sampler else None
    ms = e0.elapsed_time(e1)
    t = torch.tensor([ms], dtype=torch.float64, device=device)
    tdist.all_reduce(t, op=tdist.ReduceOp.MAX)
    nz_t = torch.tensor([nnz_local], dtype=torch.float64, device=device)
    tdist.all_reduce(nz_t)
    par_t = torch.tensor([1.0 if parity in (True, None) else 0.0], device=device)
    tdist.all_reduce(par_t, op=tdist.ReduceOp.MIN)
    launches = ds.engine.lib.sellb_launch_count() - launches0
    if graphed:   # replays do not pass through the library's launch counter
        launches += ds.graph_launches * args.steps

    # e2e through host buffers: each rank's x slice H2D from pinned memory,
    # the distributed product, y slice D2H into pinned memory, every step
    xh = torch.from_numpy(x_all[ds.r0:ds.r1].copy()).pin_memory()
    yh = torch.empty(ds.y.numel(), dtype=ds.y.dtype).pin_memory()
    e2e_steps = max(3, min(args.steps, 200))
    for _ in range(3):
        ds.x_local.copy_(xh, non_blocking=True)
        ds.step()
        yh.copy_(ds.y, non_blocking=True)
    torch.cuda.synchronize()
    tdist.barrier()
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        ds.x_local.copy_(xh, non_blocking=True)
        ds.step()
        yh.copy_(ds.y, non_blocking=True)
        torch.cuda.synchronize()
    e2e_s = torch.tensor([(time.perf_counter() - t0) / e2e_steps], dtype=torch.float64,
                         device=device)
    tdist.all_reduce(e2e_s, op=tdist.ReduceOp.MAX)
    parts = time_parts(ds, device, max(3, min(args.steps, 50)))
    if rank == 0:
        ms_max = float(t.item())
        nnz_tot = float(nz_t.item())
        value = 2.0 * nnz_tot * args.steps / (ms_max / 1e3) / 1e9
        v_alg = algorithmic_bytes(nnz_local, n_glob, sell.n_rows_padded, sell.n_chunks,
                                  s_v=s_v)
        # x read once per rank means the owned slice + halo, not the global n_cols
        v_alg = v_alg - s_v * n_glob + s_v * (n_rows_local + ds.plan.halo_entries())
        per_step_ms = ms_max / args.steps
        line = {
            "metric": args.metric, "value": round(value, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(per_step_ms, 5), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": args.dtype, "data": "synthetic",
            "config": args.config_dict,
            "details": {"nnz": int(nnz_tot), "rank0_rows": [int(ds.r0), int(ds.r1)],
                        "interior_ranges": len(ds.interior),
                        "boundary_ranges": len(ds.boundary), "build_s": round(build_s, 3),
                        "parity_vs_oracle_all_ranks": bool(par_t.item() == 1.0),
                        "parity_scope": ("each rank: its first and last 65536 rows, y "
                                         "bit-exact vs the oracle with the full x"
                                         if crs is None else
                                         "each rank: its whole slab, y bit-exact"),
                        "step_graph": graphed},
            "halo": dict(parts, **{"note": "max over ranks; exchange = NCCL send/recv post "
                                           "+ wait alone, interior / boundary = those "
                                           "chunk launches alone, eager, CUDA events"}),
            "roofline": {"bound": "hbm", "achieved": round(v_alg / (per_step_ms / 1e3) / 1e9, 2),
                         "peak": args.peak, "unit": "GB/s",
                         "frac": round(v_alg / (per_step_ms / 1e3) / 1e9 / args.peak, 4),
                         "traffic": None, "bytes_alg_per_launch": v_alg,
                         "note": "per GPU, step time = max over ranks incl. exchange"},
            "e2e": {"value": round(2.0 * nnz_tot / float(e2e_s.item()) / 1e9, 3),
                    "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(s_v * n_glob),
                    "d2h_bytes_per_step": int(s_v * sell.n_rows_padded * world),
                    "note": "per-rank pinned x slice in / y slice out each step, max over ranks"},
            "cpu_baseline": None,
            "clocks": clk,
            "gpu_launches": int(launches),
        }
        import sys
        sys.stdout.flush()
        os.write(json_fd, (json.dumps(line) + "\n").encode())
    ds.release()
    torch.cuda.synchronize()
    tdist.destroy_process_group()
    return 0
