"""Timing harness, drop-in for ``sellkit.bench``
(/root/reference/pkg/src/sellkit/bench.py:15-103).

``bench_spmv`` keeps the reference's contract -- one warm-up, ``trials`` x
``repetitions`` timed multiplications, best and median, flops = 2 nnz with
padding excluded, checksum = sum(y) -- but times on the device: x and y are
resident in HBM and each trial is bracketed by CUDA events on the launching
stream.  An injected ``timer`` switches to host wall-clock timing of the
host-array API (the reference's mode, used by deterministic tests).

Extra fields report the B200 measurement: algorithmic bytes per SpMV and the
achieved GB/s against them.
"""

import statistics
import time
from dataclasses import dataclass

import numpy as np

from . import _lib, backend
from .errors import ParameterError
from .formats import CRSMatrix, SellMatrix
from .model import algorithmic_bytes, value_bytes
from .spmv import SCHEDULINGS, spmv_crs, spmv_crs_unrolled, spmv_sell


@dataclass
class SpmvRun:
    flops: int
    wall_seconds: float
    repetitions: int
    gflops: float
    scheduling: str
    wall_seconds_median: float
    gflops_median: float
    checksum: float
    threads: int
    backend: str
    bytes_alg: int = 0
    gbps: float = 0.0
    timed_on: str = "device"


def choose_scheduling(stats, llc_bytes):
    """static if the working set fits the LLC or zeta < 0.4, else guided1
    (bench.py:35-42).  On the GPU both map to the same single launch."""
    if llc_bytes <= 0:
        raise ParameterError(f"llc_bytes must be positive, got {llc_bytes}")
    if stats.footprint_bytes <= llc_bytes or stats.zeta < 0.4:
        return "static"
    return "guided1"


def _check(repetitions, trials, scheduling):
    if repetitions < 1:
        raise ParameterError(f"repetitions must be >= 1, got {repetitions}")
    if trials < 1:
        raise ParameterError(f"trials must be >= 1, got {trials}")
    if scheduling not in SCHEDULINGS:
        raise ParameterError(f"scheduling must be one of {SCHEDULINGS}, got {scheduling!r}")


def bench_spmv(m, x, repetitions, scheduling="static", threads=1, trials=3,
               unrolled=False, timer=None, kernels=None):
    _check(repetitions, trials, scheduling)
    k = kernels or backend.kernels()
    if isinstance(m, SellMatrix):
        if unrolled:
            raise ParameterError("the unrolled kernel variant applies to CRS only")
        mult, n_out = spmv_sell, m.n_rows_padded
    elif isinstance(m, CRSMatrix):
        mult, n_out = (spmv_crs_unrolled if unrolled else spmv_crs), m.n_rows
    elif hasattr(m, "cs") and hasattr(m, "cl"):     # a reference SellMatrix
        if unrolled:
            raise ParameterError("the unrolled kernel variant applies to CRS only")
        mult, n_out = spmv_sell, m.n_rows_padded
    else:
        raise ParameterError(f"cannot benchmark a {type(m).__name__}")
    flops = 2 * m.nnz
    dt = getattr(m, "dtype", np.dtype(np.float64))
    is_sell = mult is spmv_sell
    v_alg = 0
    if is_sell:
        v_alg = algorithmic_bytes(m.nnz, m.n_cols, m.n_rows_padded, m.n_chunks,
                                  s_v=value_bytes(dt))

    device_path = (timer is None and k is backend.cuda_kernels()
                   and isinstance(m, SellMatrix))
    if not device_path:
        clock = timer or time.perf_counter
        xh = np.ascontiguousarray(x, dtype=dt)
        y = np.zeros(n_out, dtype=dt)
        mult(m, xh, y, accumulate=False, threads=threads, scheduling=scheduling, kernels=k)
        times = []
        for _ in range(trials):
            t0 = clock()
            for _ in range(repetitions):
                mult(m, xh, y, accumulate=False, threads=threads,
                     scheduling=scheduling, kernels=k)
            times.append(max(clock() - t0, 1e-12))
        checksum = float(np.sum(y))
        timed_on = "host"
    else:
        import torch
        dev = torch.device("cuda", m.device)
        tdt = torch.float32 if dt == np.float32 else torch.float64
        xd = torch.as_tensor(np.ascontiguousarray(x, dtype=dt)).to(dev)
        yd = torch.zeros(n_out, dtype=tdt, device=dev)
        lib = _lib.load()
        handle = m.handle
        with torch.cuda.device(dev):
            st = torch.cuda.current_stream()
            sp = st.cuda_stream

            def launch():
                _lib.check(lib.sellb_spmv(handle, xd.data_ptr(), yd.data_ptr(), 0,
                                          m.n_chunks, 0, _lib.ORDER_STORED, sp))
            launch()
            torch.cuda.synchronize()
            times = []
            for _ in range(trials):
                e0 = torch.cuda.Event(enable_timing=True)
                e1 = torch.cuda.Event(enable_timing=True)
                e0.record(st)
                for _ in range(repetitions):
                    launch()
                e1.record(st)
                e1.synchronize()
                times.append(max(e0.elapsed_time(e1) / 1e3, 1e-12))
            checksum = float(yd.double().sum().item())
        timed_on = "device"
    best = min(times)
    med = statistics.median(times)
    return SpmvRun(
        flops=flops, wall_seconds=best, repetitions=repetitions,
        gflops=flops * repetitions / best / 1e9, scheduling=scheduling,
        wall_seconds_median=med, gflops_median=flops * repetitions / med / 1e9,
        checksum=checksum, threads=threads, backend=k.NAME, bytes_alg=v_alg,
        gbps=v_alg * repetitions / best / 1e9 if v_alg else 0.0, timed_on=timed_on)
