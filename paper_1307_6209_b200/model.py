"""Performance model: the paper's code balance / roofline (drop-in for
``sellkit.model``, /root/reference/pkg/src/sellkit/model.py) plus the B200
measurement layer -- algorithmic bytes, the precision- and pad-skip-aware
generalised balance, and alpha recovered from measured DRAM bytes.

Paper model (fp64 values, int32 indices; model.py:5-6):
    B_CRS  = 6 + 4*alpha + 8/N_nzr                      (model.py:48-54)
    B_SELL = 6/beta + 4*alpha + 8/N_nzr                 (model.py:57-68)
    P      = b / B                                      (model.py:71-85)
    P_bar  = b * beta / 6                               (model.py:101-110)
    alpha  = (V/(2 nnz) - 6/beta - 8/N_nzr) / 4         (model.py:124-142)

Generalised (s_v value bytes, s_i index bytes, beta_eff = sector occupancy of
the pad-skipping kernel):
    B = (s_v + s_i) / (2 beta_eff) + s_v*alpha/2 + s_v/N_nzr   (+ s_v/N_nzr accumulating)
which reduces to B_SELL at s_v=8, s_i=4, beta_eff=beta.

Algorithmic bytes of one SpMV (the roofline numerator):
    V_alg = (s_v+s_i)*nnz + s_v*n_cols + s_v*N_pad + 12*n_chunks
matrix entries without padding, x read once, y written once, cs+cl.
"""

from dataclasses import dataclass

from .errors import ParameterError


@dataclass
class ModelParams:
    """alpha (RHS bytes factor), beta (chunk occupancy), N_nzr, N_nzc and the
    attainable bandwidth b in GB/s (model.py:14-38)."""

    alpha: float
    beta: float
    n_nzr: float
    n_nzc: float
    bandwidth_GBps: float

    def __post_init__(self):
        if self.alpha < 0:
            raise ParameterError(f"alpha must be >= 0, got {self.alpha}")
        if not 0.0 < self.beta <= 1.0:
            raise ParameterError(f"beta must be in (0, 1], got {self.beta}")
        if self.n_nzr <= 0:
            raise ParameterError(f"n_nzr must be positive, got {self.n_nzr}")
        if self.n_nzc <= 0:
            raise ParameterError(f"n_nzc must be positive, got {self.n_nzc}")
        if self.bandwidth_GBps <= 0:
            raise ParameterError(
                f"bandwidth_GBps must be positive, got {self.bandwidth_GBps}")


@dataclass
class ModelResult:
    code_balance_bytes_per_flop: float
    predicted_gflops: float
    caveat: str = None


@dataclass
class AlphaEstimate:
    """alpha with its plausibility flag: in_range iff 0 <= alpha <= L_C
    (L_C = line_bytes / s_v, every access misses) (model.py:113-121)."""

    alpha: float
    l_c: float
    in_range: bool


def _check_beta(beta):
    if not 0.0 < beta <= 1.0:
        raise ParameterError(f"beta must be in (0, 1], got {beta}")


def _check_nzr(n_nzr):
    if n_nzr <= 0:
        raise ParameterError(f"n_nzr must be positive, got {n_nzr}")


def _check_alpha(alpha):
    if alpha < 0:
        raise ParameterError(f"alpha must be >= 0, got {alpha}")


def code_balance_crs(alpha, n_nzr):
    """Bytes per flop of the CRS kernel: 6 + 4 alpha + 8/N_nzr."""
    _check_nzr(n_nzr)
    _check_alpha(alpha)
    return 6.0 + 4.0 * alpha + 8.0 / n_nzr


def code_balance_sell(alpha, beta, n_nzr):
    """Bytes per flop of the SELL kernel: 6/beta + 4 alpha + 8/N_nzr."""
    _check_beta(beta)
    _check_nzr(n_nzr)
    _check_alpha(alpha)
    return 6.0 / beta + 4.0 * alpha + 8.0 / n_nzr


def roofline(params, balance=None, caveat=None):
    """Predicted GF/s = b / B (B from code_balance_sell when omitted)."""
    if balance is None:
        balance = code_balance_sell(params.alpha, params.beta, params.n_nzr)
    if balance <= 0:
        raise ParameterError(f"code balance must be positive, got {balance}")
    return ModelResult(balance, params.bandwidth_GBps / balance, caveat)


def roofline_ideal_alpha(params, caveat=None):
    """Prediction with perfect RHS reuse, alpha = 1/N_nzc."""
    p = ModelParams(1.0 / params.n_nzc, params.beta, params.n_nzr, params.n_nzc,
                    params.bandwidth_GBps)
    return roofline(p, caveat=caveat)


def roofline_upper_bound(bandwidth_GBps, beta):
    """Matrix-data floor P_bar = b*beta/6 GF/s."""
    if bandwidth_GBps <= 0:
        raise ParameterError(f"bandwidth_GBps must be positive, got {bandwidth_GBps}")
    _check_beta(beta)
    return bandwidth_GBps * beta / 6.0


def infer_alpha(v_meas_bytes, n_nz, beta, n_nzr, line_bytes=64):
    """alpha = (V/(2 nnz) - 6/beta - 8/N_nzr)/4 with in_range flag."""
    if n_nz <= 0:
        raise ParameterError(f"n_nz must be positive, got {n_nz}")
    _check_beta(beta)
    _check_nzr(n_nzr)
    if line_bytes < 8:
        raise ParameterError(f"line_bytes must be >= 8, got {line_bytes}")
    alpha = (v_meas_bytes / (2.0 * n_nz) - 6.0 / beta - 8.0 / n_nzr) / 4.0
    l_c = line_bytes / 8.0
    return AlphaEstimate(alpha, l_c, bool(0.0 <= alpha <= l_c))


# ---------------------------------------------------------------------------
# B200 measurement layer
# ---------------------------------------------------------------------------

def value_bytes(dtype):
    return 4 if str(dtype) in ("float32", "f32", "fp32") else 8


def algorithmic_bytes(nnz, n_cols, n_rows_padded, n_chunks, s_v=8, s_i=4,
                      accumulate=False):
    """V_alg of one SpMV; padding excluded."""
    v = (s_v + s_i) * nnz + s_v * n_cols + s_v * n_rows_padded + 12 * n_chunks
    if accumulate:
        v += s_v * n_rows_padded
    return int(v)


def code_balance_general(alpha, beta_eff, n_nzr, s_v=8, s_i=4, accumulate=False):
    """(s_v+s_i)/(2 beta_eff) + s_v alpha/2 + s_v/N_nzr (+ s_v/N_nzr)."""
    _check_beta(beta_eff)
    _check_nzr(n_nzr)
    _check_alpha(alpha)
    b = (s_v + s_i) / (2.0 * beta_eff) + s_v * alpha / 2.0 + s_v / n_nzr
    if accumulate:
        b += s_v / n_nzr
    return b


def alpha_from_traffic(dram_bytes, nnz, matrix_bytes, n_rows_padded, n_chunks,
                       s_v=8, extra_bytes=0, line_bytes=32):
    """alpha measured from DRAM counters: the RHS share of measured traffic
    per stored entry, in units of s_v bytes.

        alpha = (dram - matrix_bytes - y - metadata - extra) / (s_v * nnz)

    ``matrix_bytes`` is what the kernel variant actually streams (all slots
    for the pad-inclusive kernel, touched sectors for the pad-skipping one);
    ``extra_bytes`` covers row_lengths / perm reads.  in_range uses
    L_C = line_bytes / s_v with B200's 32-byte sector as the line.
    """
    if nnz <= 0:
        raise ParameterError(f"nnz must be positive, got {nnz}")
    rest = dram_bytes - matrix_bytes - s_v * n_rows_padded - 12 * n_chunks - extra_bytes
    alpha = rest / (s_v * nnz)
    l_c = line_bytes / s_v
    return AlphaEstimate(alpha, l_c, bool(0.0 <= alpha <= l_c))


def roofline_fraction(v_alg_bytes, seconds, peak_GBps):
    """(V_alg / t) / peak."""
    if seconds <= 0 or peak_GBps <= 0:
        raise ParameterError("seconds and peak must be positive")
    return v_alg_bytes / seconds / 1e9 / peak_GBps
