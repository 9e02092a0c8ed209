"""Device bandwidth microbenchmarks: the B200 analog of the reference's
``membench.py`` (/root/reference/pkg/src/sellkit/membench.py:52-116), which
supplies the attainable bandwidth b for the paper's model (Listing 1
read-reduce and copy).

Both run our own kernels (``sellb_read_sum`` = 16-byte vector loads with four
partial sums per thread, ``sellb_copy``) on buffers far larger than the
126 MB L2, timed with CUDA events after a warm-up.  GB/s counts algorithmic
bytes: read = 8 n, copy = 16 n (read + write; no write-allocate on GPUs,
unlike the CPU's x1.5 factor at membench.py:21).
"""

from dataclasses import dataclass

from . import _lib


@dataclass
class MemBenchResult:
    kind: str
    bytes_per_rep: int
    seconds: float
    gbps: float


def _time(fn, reps, torch):
    fn()
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            fn()
        e1.record()
        e1.synchronize()
        best = min(best, e0.elapsed_time(e1) / 1e3 / reps)
    return best


def microbench_read_sum(n_bytes=4 << 30, reps=10, device=0):
    """Read-reduce bandwidth (membench.py:52-82)."""
    import ctypes
    import torch
    lib = _lib.require_device()
    n = n_bytes // 8
    a = torch.rand(n, dtype=torch.float64, device=f"cuda:{device}")
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.check(lib.sellb_read_sum(a.data_ptr(), n, None, st))
    t = _time(run, reps, torch)
    out = ctypes.c_double()
    _lib.check(lib.sellb_read_sum(a.data_ptr(), n, ctypes.byref(out), st))
    return MemBenchResult("read_sum", 8 * n, t, 8 * n / t / 1e9)


def microbench_copy(n_bytes=2 << 30, reps=10, device=0):
    """Copy bandwidth, read + write bytes (membench.py:85-116)."""
    import torch
    lib = _lib.require_device()
    n = n_bytes // 8
    a = torch.rand(n, dtype=torch.float64, device=f"cuda:{device}")
    b = torch.empty_like(a)
    st = torch.cuda.current_stream().cuda_stream

    def run():
        _lib.check(lib.sellb_copy(a.data_ptr(), b.data_ptr(), n, st))
    t = _time(run, reps, torch)
    return MemBenchResult("copy", 16 * n, t, 16 * n / t / 1e9)
