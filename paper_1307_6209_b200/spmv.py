"""SpMV entry points, drop-in for ``sellkit.spmv``
(/root/reference/pkg/src/sellkit/spmv.py).

``spmv_sell(m, x, y=None, accumulate=False, threads=1, scheduling="static",
kernels=None)`` keeps the reference's signature, validation and return
convention (y in stored, padded order; the caller's y object is returned).

Execution: the whole chunk range is ONE kernel launch on the GPU (one thread
per stored row).  ``threads`` and ``scheduling`` are still validated exactly
like the reference (spmv.py:20-24, 45-50) -- on the device every row has one
owner regardless, so results are bitwise independent of them, as the
reference guarantees for its thread pool.

``kernels`` selects the backend module as in the reference.  The default is
this package's CUDA module; passing another protocol module (e.g. the
reference's own compiled core) runs that module's range kernels on the host
arrays instead -- an explicit caller choice, never an automatic fallback.

Inputs may also be CUDA tensors (torch): then x/y stay on the device and
nothing crosses PCIe.
"""


import threading
import weakref

import numpy as np

from . import _lib, backend
from .errors import DimensionError, ParameterError

SCHEDULINGS = ("static", "guided1")


def _check_scheduling(scheduling):
    if scheduling not in SCHEDULINGS:
        raise ParameterError(
            f"scheduling must be one of {SCHEDULINGS}, got {scheduling!r}")


def _check_threads(threads):
    threads = int(threads)
    if threads < 1:
        raise ParameterError(f"threads must be >= 1, got {threads}")
    return threads


def _is_device_tensor(a):
    return hasattr(a, "is_cuda") and bool(a.is_cuda)


def _as_input_vector(x, n_cols, dtype=np.float64):
    x = np.ascontiguousarray(x, dtype=dtype)
    if x.ndim != 1 or len(x) != n_cols:
        raise DimensionError(f"x must be a vector of length {n_cols}")
    return x


def _as_output_vector(y, n, dtype=np.float64):
    if y is None:
        return np.zeros(n, dtype=dtype)
    if not (isinstance(y, np.ndarray) and y.dtype == dtype and y.ndim == 1
            and y.flags.c_contiguous and y.flags.writeable):
        raise ParameterError(
            f"y must be a writable contiguous {np.dtype(dtype).name} vector")
    if len(y) != n:
        raise DimensionError(f"y must have length {n}, got {len(y)}")
    return y


def _run_host_partitioned(run_range, n_units, threads, scheduling):
    """The reference's CPU work split (spmv.py:45-73) for an explicitly
    chosen host kernels module."""
    from concurrent.futures import ThreadPoolExecutor
    import threading
    if threads == 1 or n_units <= 1:
        run_range(0, n_units)
        return
    if scheduling == "static":
        b = np.linspace(0, n_units, threads + 1).astype(int)
        spans = [(int(b[t]), int(b[t + 1])) for t in range(threads) if b[t + 1] > b[t]]
        with ThreadPoolExecutor(max_workers=len(spans)) as pool:
            list(pool.map(lambda s: run_range(*s), spans))
        return
    lock, cursor = threading.Lock(), [0]

    def worker():
        while True:
            with lock:
                u = cursor[0]
                cursor[0] += 1
            if u >= n_units:
                return
            run_range(u, u + 1)

    with ThreadPoolExecutor(max_workers=threads) as pool:
        list(pool.map(lambda _: worker(), range(threads)))


# ---------------------------------------------------------------------------
# page-locking of caller vectors that come back (the iterative-solver pattern)
# ---------------------------------------------------------------------------
# A pageable NumPy vector is staged by the library through its pinned
# mirrors (host thread pool, sellb_host.cu).  A vector passed a SECOND time
# is page-locked in place instead (sellb_host_register), so later calls move
# it by DMA at pinned speed; the registration is dropped when the array is
# garbage-collected (weakref.finalize runs before NumPy frees the data).
# One-shot vectors never pay for the registration.

_PIN_MIN_BYTES = 1 << 20
_PIN_OFF = bool(__import__("os").environ.get("SELLB_NO_PIN"))   # A/B: staging only
_pin_state = {}
_pin_lock = threading.Lock()


def _data_owner(a):
    o = a
    while isinstance(o, np.ndarray) and not o.flags.owndata:
        o = o.base
    return o if isinstance(o, np.ndarray) and o.flags.owndata else None


def _unpin(key):
    with _pin_lock:
        st = _pin_state.pop(key, None)
    if st == "pinned":
        try:
            _lib.load().sellb_host_unregister(key[0])
        except Exception:          # interpreter / CUDA teardown
            pass


def _pin_hint(a):
    """Register a host vector for DMA the second time it is seen."""
    if _PIN_OFF or a.nbytes < _PIN_MIN_BYTES:
        return
    own = _data_owner(a)
    if own is None:
        return
    key = (own.ctypes.data, own.nbytes)
    with _pin_lock:
        st = _pin_state.get(key)
        if st is None:
            _pin_state[key] = "seen"
            weakref.finalize(own, _unpin, key)
            return
        if st != "seen":
            return
        rc = _lib.load().sellb_host_register(key[0], key[1])
        _pin_state[key] = "pinned" if rc == 0 else "failed"


def _device_spmv(m, x, y, accumulate, out_order, stream):
    """x, y are CUDA tensors of the matrix dtype on the matrix's device."""
    n_out = m.n_rows if out_order == _lib.ORDER_ORIGINAL else m.n_rows_padded
    if x.dim() != 1 or x.numel() != m.n_cols:
        raise DimensionError(f"x must be a vector of length {m.n_cols}")
    if y.dim() != 1 or y.numel() != n_out:
        raise DimensionError(f"y must have length {n_out}, got {y.numel()}")
    if not (x.is_contiguous() and y.is_contiguous()):
        raise ParameterError("x and y must be contiguous")
    if stream is None:
        import torch
        stream = torch.cuda.current_stream(y.device).cuda_stream
    _lib.check(_lib.load().sellb_spmv(m.handle, x.data_ptr(), y.data_ptr(), 0,
                                      m.n_chunks, int(bool(accumulate)), out_order,
                                      stream))
    return y


def spmv_sell(m, x, y=None, accumulate=False, threads=1, scheduling="static",
              kernels=None, *, out_order="stored", stream=None):
    """y (+)= m @ x for a SELL-C-sigma matrix (spmv.py:105-122).

    y is indexed by stored rows and has length n_rows_padded; use
    unpermute_vector(y, m.perm) for the original order -- or pass
    ``out_order="original"`` to get y[n_rows] unpermuted by the kernel's
    fused epilogue.  With a column-permuted matrix x is in stored-row order.
    """
    _check_scheduling(scheduling)
    threads = _check_threads(threads)
    order = {"stored": _lib.ORDER_STORED, "original": _lib.ORDER_ORIGINAL}.get(out_order)
    if order is None:
        raise ParameterError(f"out_order must be 'stored' or 'original', got {out_order!r}")
    k = kernels or backend.kernels()
    dt = getattr(m, "dtype", np.dtype(np.float64))
    if _is_device_tensor(x):
        if k is not backend.cuda_kernels():
            raise ParameterError("device tensors need the cuda kernels module")
        if y is None:
            import torch
            n_out = m.n_rows if order == _lib.ORDER_ORIGINAL else m.n_rows_padded
            y = torch.zeros(n_out, dtype=x.dtype, device=x.device)
        return _device_spmv(m, x, y, accumulate, order, stream)

    x = _as_input_vector(x, m.n_cols, dt)
    n_out = m.n_rows if order == _lib.ORDER_ORIGINAL else m.n_rows_padded
    y = _as_output_vector(y, n_out, dt)
    if k is backend.cuda_kernels() and hasattr(m, "handle"):
        lib = _lib.require_device()
        _pin_hint(x)
        _pin_hint(y)
        _lib.check(lib.sellb_spmv_host(
            m.handle, _lib.ptr(x), _lib.ptr(y), 0, m.n_chunks,
            int(bool(accumulate)), order, stream))
        return y
    if order != _lib.ORDER_STORED:
        raise ParameterError("out_order='original' needs the cuda kernels module")

    def run_range(c0, c1):
        k.spmv_sell_range(m.cs, m.cl, m.C, m.col, m.val, x, y, c0, c1, accumulate)

    if k is backend.cuda_kernels():
        run_range(0, m.n_chunks)      # one launch over every chunk
    else:
        _run_host_partitioned(run_range, m.n_chunks, threads, scheduling)
    return y


def spmv_crs(m, x, y=None, accumulate=False, threads=1, scheduling="static",
             kernels=None):
    """y (+)= m @ x for a CRS matrix (spmv.py:76-87), on the GPU."""
    _check_scheduling(scheduling)
    threads = _check_threads(threads)
    k = kernels or backend.kernels()
    x = _as_input_vector(x, m.n_cols)
    y = _as_output_vector(y, m.n_rows)

    def run_range(r0, r1):
        k.spmv_crs_range(m.rpt, m.col, m.val, x, y, r0, r1, accumulate)

    if k is backend.cuda_kernels():
        run_range(0, m.n_rows)
    else:
        _run_host_partitioned(run_range, m.n_rows, threads, scheduling)
    return y


def spmv_crs_unrolled(m, x, y=None, accumulate=False, threads=1,
                      scheduling="static", kernels=None):
    """Four partial sums per row (spmv.py:90-102, _kernels.pyx:34-62)."""
    _check_scheduling(scheduling)
    threads = _check_threads(threads)
    k = kernels or backend.kernels()
    x = _as_input_vector(x, m.n_cols)
    y = _as_output_vector(y, m.n_rows)

    def run_range(r0, r1):
        k.spmv_crs_unrolled_range(m.rpt, m.col, m.val, x, y, r0, r1, accumulate)

    if k is backend.cuda_kernels():
        run_range(0, m.n_rows)
    else:
        _run_host_partitioned(run_range, m.n_rows, threads, scheduling)
    return y



class SpmvChain:
    """The iterative-solver pattern in permuted space:
    ``steps`` products, each one's output the next one's input, entirely on
    the GPU -- x_{k+1} = A x_k for a square matrix built with
    ``permute_cols=True`` (rows and columns share the stored index space, so
    no vector is permuted between steps).

    The two vectors ping-pong in one buffer pair owned by the chain.  With
    ``graph=True`` the steps are captured once into a CUDA graph on the first
    ``run`` and replayed afterwards (one launch per run instead of
    ``steps``); the vector stays in the 126 MB L2 between steps when it fits.
    Every step is the reference's product bit for bit.
    """

    def __init__(self, m, steps, *, dtype=None, graph=True, device=0):
        import torch
        if m.n_rows != m.n_cols:
            raise ParameterError("spmv_chain needs a square matrix")
        if not getattr(m, "col_permuted", False) and m.n_rows > 1:
            raise ParameterError("spmv_chain needs permute_cols=True (stored index space)")
        if steps < 0:
            raise ParameterError("steps must be >= 0")
        self.m, self.steps, self.graph = m, int(steps), bool(graph)
        f32 = np.dtype(getattr(m, "dtype", np.float64)) == np.float32
        self.dtype = torch.float32 if f32 else torch.float64
        if dtype is not None and dtype != self.dtype:
            raise ParameterError(f"dtype {dtype} does not match the matrix")
        self.dev = torch.device("cuda", device)
        self.buf = [torch.zeros(m.n_rows_padded, dtype=self.dtype, device=self.dev)
                    for _ in range(2)]
        self.stream = torch.cuda.Stream(device=self.dev)
        self._g = None
        self._lib = _lib.require_device()

    def _run(self, k0, k1):
        st = self.stream.cuda_stream
        for k in range(k0, k1):
            src, dst = self.buf[k & 1], self.buf[(k + 1) & 1]
            _lib.check(self._lib.sellb_spmv(self.m.handle, src.data_ptr(), dst.data_ptr(), 0,
                                            self.m.n_chunks, 0, _lib.ORDER_STORED, st))

    def run(self, x):
        """x: CUDA vector of length n_rows (stored order) -> the last product
        (length n_rows_padded, a view of the chain's buffer: copy it to keep
        it past the next run)."""
        import torch
        m = self.m
        if not _is_device_tensor(x) or x.dim() != 1 or x.numel() != m.n_rows:
            raise DimensionError(f"x must be a CUDA vector of length {m.n_rows}")
        if x.dtype != self.dtype:
            raise ParameterError(f"x dtype {x.dtype} does not match the matrix")
        cur = torch.cuda.current_stream(self.dev)
        self.stream.wait_stream(cur)
        with torch.cuda.stream(self.stream):
            self.buf[0][:m.n_rows].copy_(x)
            if self.steps:
                if not self.graph or self.steps == 1:
                    self._run(0, self.steps)
                elif self._g is None:
                    self._run(0, 1)          # eager first step: lazy state, attributes
                    g = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(g, stream=self.stream):
                        self._run(1, self.steps)
                    g.replay()
                    self._g = g
                else:
                    self._run(0, 1)
                    self._g.replay()
        cur.wait_stream(self.stream)
        return self.buf[self.steps & 1]


def spmv_chain(m, x, steps, *, graph=True):
    """``steps`` chained products x_{k+1} = A x_k in permuted space
    (SpmvChain for repeated use); returns a new tensor."""
    ch = SpmvChain(m, steps, dtype=x.dtype if _is_device_tensor(x) else None, graph=graph,
                   device=x.device.index if _is_device_tensor(x) else 0)
    return ch.run(x).clone()
