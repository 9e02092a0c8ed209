"""Deterministic synthetic matrices.

Two groups:

* the reference's generators (/root/reference/pkg/src/sellkit/generate.py),
  same signatures and returned COO: gen_worst_case, gen_dense, gen_banded,
  gen_skewed;
* the BASELINE.json configurations, built straight into CRS with vectorised
  NumPy (the reference has no generator for them):
    cfg1  laplace2d(1000)          2D 5-point Laplacian, N=1e6, nnz=4,996,000
    cfg2  stencil27(128)           3D 27-point stencil, N=2,097,152, nnz=55,742,968
    cfg3  powerlaw(4_000_000)      Pareto row lengths, mean ~20, zeta ~2
    cfg4  gen_skewed(2**21, 8, 2048, 1024)
    cfg5  hamiltonian(2**26)       banded-random, ~19.4 nnz/row (row-addressable)

The same CRS feeds the CPU oracle and the GPU, so parity is on identical
inputs.  ``rhs(n)`` is the reference CLI's x (cli.py:35,174-175).
"""

import numpy as np

from .errors import ParameterError
from .formats import COOMatrix, CRSMatrix, OFFSET_DTYPE, canonicalize_coo

X_SEED = 12345


def rhs(n_cols, seed=X_SEED, dtype=np.float64):
    """x = default_rng(12345).uniform(-1, 1, n_cols) (cli.py:174-175)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n_cols).astype(dtype)


# ---------------------------------------------------------------------------
# reference generators (generate.py:13-96)
# ---------------------------------------------------------------------------

def gen_worst_case(n_chunks, C, seed=0):
    """One full row leading every block of C rows, the rest diagonal-only:
    beta(sigma=1) = (N+C-1)/(C N), sigma = C^2 sorts it to 1."""
    if n_chunks < 1:
        raise ParameterError(f"n_chunks must be >= 1, got {n_chunks}")
    if C < 2:
        raise ParameterError(f"C must be >= 2, got {C}")
    n = n_chunks * C
    full = np.arange(n_chunks, dtype=OFFSET_DTYPE) * C
    single = np.setdiff1d(np.arange(n, dtype=OFFSET_DTYPE), full)
    rows = np.concatenate([np.repeat(full, n), single])
    cols = np.concatenate([np.tile(np.arange(n, dtype=OFFSET_DTYPE), n_chunks), single])
    vals = np.random.default_rng(seed).uniform(0.1, 1.0, size=len(rows))
    return canonicalize_coo(COOMatrix(n, n, rows, cols, vals))


def gen_dense(n, seed=0):
    if n < 1:
        raise ParameterError(f"n must be >= 1, got {n}")
    rows = np.repeat(np.arange(n, dtype=OFFSET_DTYPE), n)
    cols = np.tile(np.arange(n, dtype=OFFSET_DTYPE), n)
    return COOMatrix(n, n, rows, cols,
                     np.random.default_rng(seed).uniform(0.1, 1.0, size=n * n))


def gen_banded(n, half_bw, fill=1.0, seed=0):
    if n < 1:
        raise ParameterError(f"n must be >= 1, got {n}")
    if half_bw < 0 or half_bw >= n:
        raise ParameterError(f"half_bw must be in [0, n), got {half_bw}")
    if not 0.0 < fill <= 1.0:
        raise ParameterError(f"fill must be in (0, 1], got {fill}")
    w = 2 * half_bw + 1
    i = np.repeat(np.arange(n, dtype=OFFSET_DTYPE), w)
    j = i + np.tile(np.arange(-half_bw, half_bw + 1, dtype=OFFSET_DTYPE), n)
    keep = (j >= 0) & (j < n)
    if fill < 1.0:
        keep &= (np.random.default_rng(seed + 1).random(len(j)) < fill) | (i == j)
    rows, cols = i[keep], j[keep]
    vals = np.random.default_rng(seed).uniform(0.1, 1.0, size=len(rows))
    return COOMatrix(n, n, rows, cols, vals)


def gen_skewed(n, base_len, spike_len, spike_count, seed=0):
    if n < 1:
        raise ParameterError(f"n must be >= 1, got {n}")
    if not 1 <= base_len <= n:
        raise ParameterError(f"base_len must be in [1, n], got {base_len}")
    if not 1 <= spike_len <= n:
        raise ParameterError(f"spike_len must be in [1, n], got {spike_len}")
    if not 0 <= spike_count <= n:
        raise ParameterError(f"spike_count must be in [0, n], got {spike_count}")
    lengths = np.full(n, base_len, dtype=OFFSET_DTYPE)
    if spike_count:
        lengths[np.unique(np.linspace(0, n - 1, spike_count).astype(OFFSET_DTYPE))] = spike_len
    rows = np.repeat(np.arange(n, dtype=OFFSET_DTYPE), lengths)
    first = np.cumsum(lengths) - lengths
    k = np.arange(int(lengths.sum()), dtype=OFFSET_DTYPE) - np.repeat(first, lengths)
    cols = (rows + k) % n
    vals = np.random.default_rng(seed).uniform(0.1, 1.0, size=len(rows))
    return canonicalize_coo(COOMatrix(n, n, rows, cols, vals))


# ---------------------------------------------------------------------------
# BASELINE configurations (CRS directly)
# ---------------------------------------------------------------------------

def _stencil(shape, offsets, diag, off, rows=None):
    """CRS of a constant-coefficient stencil on a row-major grid with
    Dirichlet truncation.  Offsets are visited in increasing linear offset,
    so columns ascend inside every row.  ``rows=(r0, r1)`` builds only that
    row block (global column indices), for the row-partitioned runs."""
    shape = tuple(int(s) for s in shape)
    n_glob = int(np.prod(shape))
    r0, r1 = (0, n_glob) if rows is None else (int(rows[0]), int(rows[1]))
    n = r1 - r0
    strides = np.cumprod((1,) + shape[::-1][:-1])[::-1]
    offsets = sorted(offsets, key=lambda o: int(np.dot(o, strides)))
    coords = np.array(np.unravel_index(np.arange(r0, r1), shape), dtype=np.int32)
    k = len(offsets)
    mask = np.ones((n, k), dtype=bool)
    lin = np.empty(k, dtype=np.int64)
    for t, o in enumerate(offsets):
        for d, od in enumerate(o):
            if od:
                c = coords[d] + od
                mask[:, t] &= (c >= 0) & (c < shape[d])
        lin[t] = int(np.dot(o, strides))
    counts = mask.sum(axis=1)
    rpt = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(counts, out=rpt[1:])
    rr, tt = np.nonzero(mask)
    col = (rr + r0 + lin[tt]).astype(np.int32)
    is_diag = lin[tt] == 0
    val = np.where(is_diag, diag, off).astype(np.float64)
    return CRSMatrix(n, n_glob, rpt, col, val)


def laplace2d(nx=1000):
    """cfg1: 5-point Laplacian, diag 4, neighbours -1 (nnz = 5N - 4 nx)."""
    offs = [(0, 0), (-1, 0), (1, 0), (0, -1), (0, 1)]
    return _stencil((nx, nx), offs, 4.0, -1.0)


def stencil27(n=128, nz=None):
    """cfg2: 27-point stencil on n x n x nz (nz defaults to n), diag 26,
    others -1.  Grid index order (z, y, x), x fastest."""
    nz = n if nz is None else nz
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    return _stencil((nz, n, n), offs, 26.0, -1.0)


def stencil27_slab(n, nz_total, z0, z1):
    """Rows of z-planes [z0, z1) of the 27-point stencil on n x n x nz_total,
    with global column indices (one GPU's block of the weak-scaling run)."""
    offs = [(a, b, c) for a in (-1, 0, 1) for b in (-1, 0, 1) for c in (-1, 0, 1)]
    return _stencil((nz_total, n, n), offs, 26.0, -1.0, rows=(z0 * n * n, z1 * n * n))


def _splitmix64(z):
    z = (z + np.uint64(0x9E3779B97F4A7C15)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    z = ((z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    z = ((z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)) & np.uint64(0xFFFFFFFFFFFFFFFF)
    return z ^ (z >> np.uint64(31))


_M64 = (1 << 64) - 1


def _pl_lengths(rows, n, mean_base, lmax, seed):
    su = np.uint64((seed * 0xA24BAED4963EE407) & _M64)
    hu = _splitmix64(rows.astype(np.uint64) ^ su)
    u = (hu >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    q = mean_base / np.sqrt(1.0 - u)
    return np.clip(np.floor(q), 1, min(lmax, n)).astype(np.int64)


def powerlaw_rows(n, r0, r1, mean_base=10.0, lmax=4096, band=50_000, seed=3):
    """Rows [r0, r1) of the cfg3 power-law matrix, row-addressable (any
    block regenerates alone; the device generator, csrc/sellb_gen.cu
    k_pl_*, is bit-identical).  Row i: length floor(mean_base / sqrt(1 - u_i))
    clipped to [1, min(lmax, n)] with u_i a counter hash in [0, 1) -- the
    inverse CDF of mean_base (1 + Pareto(2)), mean ~20, zeta ~2; columns one
    contiguous window starting at a hashed offset within +-band of the
    diagonal; values counter hashes mapped to [-1, 1), exact in fp64."""
    rows = np.arange(r0, r1, dtype=np.int64)
    lengths = _pl_lengths(rows, n, mean_base, lmax, seed)
    h = _splitmix64(rows.astype(np.uint64) ^ np.uint64(seed))
    start = rows + (h % np.uint64(2 * band + 1)).astype(np.int64) - band
    start = np.clip(np.minimum(start, n - lengths), 0, None)
    rpt = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(lengths, out=rpt[1:])
    nnz = int(rpt[-1])
    k = np.arange(nnz, dtype=np.int64) - np.repeat(rpt[:-1], lengths)
    col = (np.repeat(start, lengths) + k).astype(np.int32)
    rk = np.repeat(rows.astype(np.uint64) * np.uint64(0x100000001B3), lengths)
    vh = _splitmix64(rk ^ (k.astype(np.uint64) +
                           np.uint64((seed + 0x5851F42D4C957F2D) & _M64)))
    val = (vh >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0
    return rpt, col, val


def powerlaw(n=4_000_000, mean_base=10.0, lmax=4096, band=50_000, seed=3):
    """cfg3 (BASELINE configs[2]): N = 4M power-law rows, see powerlaw_rows."""
    with np.errstate(over="ignore"):
        rpt, col, val = powerlaw_rows(n, 0, n, mean_base, lmax, band, seed)
    return CRSMatrix(n, n, rpt, col, val)


def powerlaw_device(n=4_000_000, r0=0, r1=None, mean_base=10.0, lmax=4096, band=50_000,
                    seed=3, device=0, dtype=np.float64):
    """Rows [r0, r1) of the cfg3 matrix generated ON the GPU (bit-identical to
    powerlaw_rows).  Returns torch CUDA tensors (rpt, col, val)."""
    import ctypes
    import torch
    from . import _lib
    r1 = n if r1 is None else r1
    lib = _lib.require_device()
    dev = torch.device("cuda", device)
    rpt = torch.empty(r1 - r0 + 1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    nnz = ctypes.c_int64(0)
    with torch.cuda.device(dev):
        _lib.check(lib.sellb_gen_powerlaw_rpt(n, r0, r1, float(mean_base), int(lmax),
                                              int(seed), rpt.data_ptr(), ctypes.byref(nnz), st))
        f32 = np.dtype(dtype) == np.float32
        col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
        val = torch.empty(max(nnz.value, 1), dtype=torch.float32 if f32 else torch.float64,
                          device=dev)
        _lib.check(lib.sellb_gen_powerlaw_fill(
            n, r0, r1, float(mean_base), int(lmax), int(band), int(seed), rpt.data_ptr(),
            col.data_ptr(), val.data_ptr(), _lib.SELLB_F32 if f32 else _lib.SELLB_F64, st))
    return rpt, col[: nnz.value], val[: nnz.value]


# cfg5 hopping offsets: short bands plus long-range hops (|d| up to N/16);
# each off-diagonal kept with a hashed probability.  The offsets set the
# halo volume of the row-partitioned run.
HAM_OFFSETS = (1, 2, 3, 4, 8, 16, 64, 256, 1024, 4096, 65536, 1 << 20)


def hamiltonian_rows(n, r0, r1, keep=0.78, seed=11, offsets=HAM_OFFSETS):
    """Rows [r0, r1) of the cfg5 banded-random matrix, row-addressable: entry
    (i, i+d) exists iff hash(seed, i, d) < keep (d = 0 always); the value is
    a counter hash mapped to (-1, 1) exactly representable in fp64.  Any
    block can be regenerated alone (block-wise parity at 1.3e9 nnz)."""
    offs = np.array(sorted({0} | {d for d in offsets if d < n} |
                           {-d for d in offsets if d < n}), dtype=np.int64)
    rows = np.arange(r0, r1, dtype=np.int64)
    cols = rows[:, None] + offs[None, :]
    key = (rows[:, None].astype(np.uint64) * np.uint64(0x100000001B3)) ^ \
        (offs[None, :].astype(np.uint64) + np.uint64(seed))
    h = _splitmix64(key)
    u = (h >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
    mask = (cols >= 0) & (cols < n) & ((u < keep) | (offs[None, :] == 0))
    counts = mask.sum(axis=1)
    rpt = np.zeros(len(rows) + 1, dtype=np.int64)
    np.cumsum(counts, out=rpt[1:])
    vh = _splitmix64(h ^ np.uint64(0xD1B54A32D192ED03))
    vals = (vh >> np.uint64(11)).astype(np.float64) * (2.0 / 9007199254740992.0) - 1.0
    return rpt, cols[mask].astype(np.int32), vals[mask]


def hamiltonian(n=1 << 26, **kw):
    rpt, col, val = hamiltonian_rows(n, 0, n, **kw)
    return CRSMatrix(n, n, rpt, col, val)


CONFIGS = {
    "cfg1": lambda: laplace2d(1000),
    "cfg2": lambda: stencil27(128),
    "cfg3": lambda: powerlaw(4_000_000),
    "cfg4": lambda: canonical_crs(gen_skewed(1 << 21, 8, 2048, 1024)),
}


def canonical_crs(coo):
    from .formats import coo_to_crs
    return coo_to_crs(coo)


def hamiltonian_offsets(n, offsets=HAM_OFFSETS):
    """The sorted offset set of hamiltonian_rows (d = 0 plus +-d, |d| < n)."""
    return np.array(sorted({0} | {d for d in offsets if d < n} | {-d for d in offsets if d < n}),
                    dtype=np.int64)


def hamiltonian_device(n=1 << 26, r0=0, r1=None, keep=0.78, seed=11, device=0,
                       dtype=np.float64, offsets=HAM_OFFSETS):
    """Rows [r0, r1) of the cfg5 matrix generated ON the GPU (CUDA kernels in
    csrc/sellb_gen.cu, bit-identical to hamiltonian_rows).  Returns torch
    CUDA tensors (rpt int64[rows+1], col int32[nnz], val f64/f32[nnz]) --
    the 1.3e9-nonzero matrix never exists in host memory."""
    import ctypes
    import torch
    from . import _lib
    r1 = n if r1 is None else r1
    lib = _lib.require_device()
    dev = torch.device("cuda", device)
    offs = torch.from_numpy(hamiltonian_offsets(n, offsets)).to(dev)
    rows = r1 - r0
    rpt = torch.empty(rows + 1, dtype=torch.int64, device=dev)
    st = torch.cuda.current_stream(dev).cuda_stream
    nnz = ctypes.c_int64(0)
    with torch.cuda.device(dev):
        _lib.check(lib.sellb_gen_hamiltonian_rpt(n, r0, r1, offs.data_ptr(), offs.numel(),
                                                 keep, seed, rpt.data_ptr(),
                                                 ctypes.byref(nnz), st))
        col = torch.empty(max(nnz.value, 1), dtype=torch.int32, device=dev)
        f32 = np.dtype(dtype) == np.float32
        val = torch.empty(max(nnz.value, 1), dtype=torch.float32 if f32 else torch.float64,
                          device=dev)
        _lib.check(lib.sellb_gen_hamiltonian_fill(
            n, r0, r1, offs.data_ptr(), offs.numel(), keep, seed, rpt.data_ptr(),
            col.data_ptr(), val.data_ptr(), _lib.SELLB_F32 if f32 else _lib.SELLB_F64, st))
    return rpt, col[: nnz.value], val[: nnz.value]
