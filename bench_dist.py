"""Multi-GPU leg of bench.py (torchrun, one process per GPU, NCCL).

Lives beside bench.py, outside the product package: it uses the CPU oracle
as the parity checker for each rank's block, which the package never
imports.
"""


import numpy as np
import torch
import torch.distributed as tdist


def bench_main(args):
    """Multi-GPU benchmark under torchrun (one process per GPU, NCCL).

    cfg2 (default) -- weak scaling: the 27-point stencil on 128 x 128 x
    (128 N), one 128^3 z-slab per GPU, halo = one 128x128 plane per
    neighbour.  cfg5 -- strong scaling: the N = 2^26 banded-random matrix
    split into N row blocks, each generated and built on its own GPU, halo
    over the +-2^20 hops."""
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
    rank = int(os.environ["RANK"])
    world = int(os.environ["WORLD_SIZE"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    device = torch.device("cuda", local)
    tdist.init_process_group("nccl", device_id=device)
    C, sigma = 32, args.sigma
    t0 = time.perf_counter()
    if args.config == "cfg5":
        n_glob = args.n or (1 << 26)
        bounds = _cfg5_bounds(n_glob, world, C, sigma)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        rpt_t, col_t, val_t = generate.hamiltonian_device(n_glob, r0, r1, device=local)
        ds = setup_device(rpt_t, col_t, val_t, n_glob, bounds, C, sigma, rank, world, device)
        del rpt_t, col_t, val_t
        torch.cuda.empty_cache()
        workload = (f"banded-random N={n_glob} (device-generated) in {world} row blocks, "
                    f"SELL-32-{sigma}, NCCL halo")
        scaling = "strong"
        crs = None
    else:
        n, nz_per = 128, 128
        nz = nz_per * world
        n_glob = n * n * nz
        crs = generate.stencil27_slab(n, nz, rank * nz_per, (rank + 1) * nz_per)
        bounds = np.arange(world + 1, dtype=np.int64) * (n * n * nz_per)
        ds = setup(crs, bounds, C, sigma, rank, world, device,
                   cuda_engine_factory(C, sigma, device))
        workload = (f"3D 27-point stencil 128x128x{nz} row-partitioned into {world} "
                    f"z-slabs, SELL-32-{sigma}, NCCL halo")
        scaling = "weak"
    torch.cuda.synchronize()
    build_s = time.perf_counter() - t0
    x_glob_rng = np.random.default_rng(12345)
    x_all = x_glob_rng.uniform(-1, 1, n_glob)
    ds.x_local.copy_(torch.from_numpy(x_all[ds.r0:ds.r1]))
    sell = ds.engine.sell
    nnz_local = sell.nnz
    n_rows_local = ds.r1 - ds.r0
    # parity of this rank's block (cfg5: its first 65536 rows) against the
    # oracle with the full x -- block builds equal slices
    parity = None
    if not args.skip_parity:
        import oracle
        ds.step()
        torch.cuda.synchronize()
        if crs is None:
            from paper_1307_6209_b200.formats import CRSMatrix
            blk = min(1 << 16, n_rows_local)
            rp, cl_, vl = generate.hamiltonian_rows(n_glob, ds.r0, ds.r0 + blk)
            crs_chk = CRSMatrix(blk, n_glob, rp, cl_, vl)
        else:
            crs_chk = crs
        o = oracle.crs_to_sell(crs_chk.rpt, crs_chk.col, crs_chk.val, crs_chk.n_rows,
                               crs_chk.n_cols, C, sigma)
        y_ref = oracle.spmv_sell(o, x_all, threads=max(1, (os.cpu_count() or 8) // world))
        parity = bool(ds.y[:len(y_ref)].cpu().numpy().tobytes() == y_ref.tobytes())
    for _ in range(args.warmup):
        ds.step()
    torch.cuda.synchronize()
    # one CUDA graph per step (NCCL post included) unless SELLB_DIST_GRAPH=0;
    # kept only if its replay is bitwise equal to the eager step on all ranks
    # (tools/dist_graph_selftest.py: NCCL P2P kernels inside the graph)
    graphed = False
    if os.environ.get("SELLB_DIST_GRAPH", "1") != "0":
        graphed = ds.capture()
        for _ in range(args.warmup):
            ds.step()
        torch.cuda.synchronize()
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
    if rank == 0:
        ms_max = float(t.item())
        nnz_tot = float(nz_t.item())
        value = 2.0 * nnz_tot * args.steps / (ms_max / 1e3) / 1e9
        v_alg = algorithmic_bytes(nnz_local, n_glob, sell.n_rows_padded, sell.n_chunks)
        # x read once per rank means the owned slice + halo, not the global n_cols
        v_alg = v_alg - 8 * n_glob + 8 * (n_rows_local + ds.plan.halo_entries())
        per_step_ms = ms_max / args.steps
        line = {
            "metric": "spMVM GFLOP/s (2*nnz/t), fp64 SELL-C-sigma", "value": round(value, 3),
            "unit": "GFLOP/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": round(per_step_ms, 5), "higher_is_better": True,
            "scaling": scaling, "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload,
                       "parallelism": f"row-blocks x{world}", "nnz": int(nnz_tot),
                       "halo_bytes_per_rank": ds.plan.bytes_per_step(),
                       "interior_ranges": len(ds.interior),
                       "boundary_ranges": len(ds.boundary), "build_s": round(build_s, 3),
                       "parity_vs_oracle_all_ranks": bool(par_t.item() == 1.0),
                       "step_graph": graphed,
                       "l2": "inputs larger than L2"},
            "roofline": {"bound": "hbm", "achieved": round(v_alg / (per_step_ms / 1e3) / 1e9, 2),
                         "peak": args.peak, "unit": "GB/s",
                         "frac": round(v_alg / (per_step_ms / 1e3) / 1e9 / args.peak, 4),
                         "traffic": None, "bytes_alg_per_launch": v_alg,
                         "note": "per GPU, step time = max over ranks incl. exchange"},
            "e2e": {"value": round(2.0 * nnz_tot / float(e2e_s.item()) / 1e9, 3),
                    "unit": "GFLOP/s",
                    "h2d_bytes_per_step": int(8 * n_glob),
                    "d2h_bytes_per_step": int(8 * sell.n_rows_padded * world),
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
