"""spmv_chain: the iterative-solver loop in permuted space (PAPER.md:751-760,
SURVEY.md §8(f)4) -- k products, each feeding the next, captured in a CUDA
graph -- equals k reference products bit for bit (the CPU oracle on the
column-permuted layout, y[:n] fed back as the next x)."""

import numpy as np
import pytest

import oracle
import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import generate
from paper_1307_6209_b200.errors import DimensionError, ParameterError

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def oracle_chain(m, C, sigma, x, steps, dt):
    o = oracle.crs_to_sell(m.rpt, m.col, m.val.astype(dt), m.n_rows, m.n_cols, C, sigma,
                           1, True)
    v = x.copy()
    y = v
    for _ in range(steps):
        y = oracle.spmv_sell(o, v)
        v = y[:m.n_rows].copy()
    return y


def scaled(m, s):
    return sb.CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val * s)


@pytest.mark.parametrize("graph", [True, False])
@pytest.mark.parametrize("dt", [np.float64, np.float32])
@pytest.mark.parametrize("kind,C,sigma", [("stencil", 32, 1), ("stencil", 8, 64),
                                          ("powerlaw", 32, 10**9), ("powerlaw", 32, 128)])
def test_chain_bitwise(kind, C, sigma, dt, graph):
    import torch
    if kind == "stencil":
        m = scaled(generate.stencil27(20), 1.0 / 27)
    else:
        m = generate.powerlaw(30_000, lmax=600, band=3000, seed=5)
        m = scaled(m, 1.0 / 40)
    s = sb.crs_to_sell(m, C, sigma, permute_cols=True, dtype=dt)
    x = generate.rhs(m.n_cols).astype(dt)
    steps = 13
    xp = sb.permute_vector(x, s.perm).astype(dt)          # original -> stored order
    want = oracle_chain(m, C, sigma, xp, steps, dt)
    xs = torch.from_numpy(xp.copy()).cuda()
    got = sb.spmv_chain(s, xs, steps, graph=graph).cpu().numpy()
    assert got.tobytes() == want.tobytes()


def test_chain_zero_and_one_step():
    import torch
    m = scaled(generate.stencil27(12), 1.0 / 27)
    s = sb.crs_to_sell(m, 32, 1, permute_cols=True)
    x = torch.from_numpy(generate.rhs(m.n_cols)).cuda()
    z = sb.spmv_chain(s, x, 0)
    assert np.array_equal(z[:m.n_rows].cpu().numpy(), x.cpu().numpy())
    one = sb.spmv_chain(s, x, 1).cpu().numpy()
    assert one.tobytes() == sb.spmv_sell(s, x).cpu().numpy().tobytes()


def test_chain_argument_errors():
    import torch
    m = generate.stencil27(8)
    s = sb.crs_to_sell(m, 32, 1)                        # not column-permuted
    x = torch.zeros(m.n_rows, dtype=torch.float64, device="cuda")
    with pytest.raises(ParameterError):
        sb.spmv_chain(s, x, 3)
    sp = sb.crs_to_sell(m, 32, 1, permute_cols=True)
    with pytest.raises(DimensionError):
        sb.spmv_chain(sp, x[:-1], 3)
    with pytest.raises(ParameterError):
        sb.spmv_chain(sp, x.float(), 3)
