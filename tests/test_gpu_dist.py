"""The row-partitioned path's CUDA pieces on ONE GPU: every virtual rank's
block is built and multiplied by its own CudaEngine; the halo exchange is a
loopback (device copies in one process, no rank waits on another).  Each
block's y must equal the single-GPU product bit for bit."""

import numpy as np
import pytest
import torch

import paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, dist, generate

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module", autouse=True)
def _need_gpu():
    if not sb.HAS_CUDA:
        pytest.skip("no CUDA device")


def block(m, r0, r1):
    s, e = m.rpt[r0], m.rpt[r1]
    return CRSMatrix(r1 - r0, m.n_cols, m.rpt[r0:r1 + 1] - s, m.col[s:e], m.val[s:e])


def virtual_cluster(m, world, C, sigma):
    dev = torch.device("cuda", 0)
    bounds = dist.partition_rows(m.rpt, world, C, sigma)
    blocks = [block(m, int(bounds[r]), int(bounds[r + 1])) for r in range(world)]
    make = dist.cuda_engine_factory(C, sigma, dev)
    built = [make(b) for b in blocks]
    gathered = [(dist.HaloPlan.requests(b.col, bounds, r), built[r][1]["has_padding"],
                 dist.HaloPlan.reads_x0(b.col, bounds, r)) for r, b in enumerate(blocks)]
    dss = [dist.setup(b, bounds, C, sigma, r, world, dev, None,
                      plan=dist.HaloPlan.from_requests(r, world, bounds, gathered),
                      built=built[r]) for r, b in enumerate(blocks)]
    return bounds, dss


def loopback_step(dss, x):
    """DistSpmv._step_eager with the NCCL batch replaced by device copies."""
    xt = torch.from_numpy(x).cuda()
    for ds in dss:
        ds.x_local.copy_(xt[ds.r0:ds.r1])
        if ds.x0_recv:
            ds.x_full[0:1].zero_()
    for r, ds in enumerate(dss):
        for p, buf, gidx in ds.send_ops:
            if gidx is not None:
                ds.engine.gather(ds.x_full, gidx, buf)
            dst = [ro for ro in dss[p].recv_ops if ro[0] == r][0][1]
            dst.copy_(buf)
        for p in ds.x0_peers:
            dss[p].x0_buf.copy_(ds.x_full[0:1])
    for ds in dss:
        ds.engine.run_ranges(ds.interior, ds.x_full, ds.y)
        if ds.x0_recv:
            ds.x_full[0:1].copy_(ds.x0_buf)
        for p, buf, gidx in ds.recv_ops:
            if gidx is not None:
                ds.engine.scatter(buf, gidx, ds.x_full)
        ds.engine.run_ranges(ds.boundary, ds.x_full, ds.y)
        if ds.x0_recv and ds.has_padding:
            ds.engine.pad_fixup(ds.x0_buf, ds.y)
    torch.cuda.synchronize()
    return [ds.y.cpu().numpy() for ds in dss]


@pytest.mark.parametrize("world", [2, 4, 8])
@pytest.mark.parametrize("name,C,sigma", [("stencil", 32, 1), ("powerlaw", 32, 128),
                                          ("hamiltonian", 32, 1)])
def test_blocks_equal_single_gpu(world, name, C, sigma):
    m = {"stencil": lambda: generate.stencil27(32, nz=64),
         "powerlaw": lambda: generate.powerlaw(200_000, seed=4, band=5000),
         "hamiltonian": lambda: generate.hamiltonian(1 << 18)}[name]()
    bounds, dss = virtual_cluster(m, world, C, sigma)
    for x0 in (None, np.inf):
        x = generate.rhs(m.n_cols)
        if x0 is not None:
            x[0] = x0
        ys = loopback_step(dss, x)
        for r, y in enumerate(ys):
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            ref = sb.spmv_sell(sb.crs_to_sell(block(m, r0, r1), C, sigma), x)
            if x0 is None:
                assert y.tobytes() == ref.tobytes(), (r, name)
            else:
                np.testing.assert_array_equal(y, ref)
        if x0 is None:
            full = sb.spmv_sell(sb.crs_to_sell(m, C, sigma), x)
            stitched = np.concatenate([ys[r][: int(bounds[r + 1] - bounds[r])]
                                       for r in range(world)])
            assert stitched.tobytes() == full[: m.n_rows].tobytes()


def test_cfg5_device_setup_loopback():
    """setup_device (device-resident CRS, torch-side halo plan, chunk flags
    from sellb_chunk_flags) for 4 virtual ranks of the cfg5 generator; each
    block's y equals the single-GPU product's slice."""
    n, world, C, sigma = 1 << 20, 4, 32, 512
    dev = torch.device("cuda", 0)
    bounds = dist._cfg5_bounds(n, world, C, sigma)
    blocks = [generate.hamiltonian_device(n, int(bounds[r]), int(bounds[r + 1]))
              for r in range(world)]
    gathered = [(dist.requests_torch(b[1], bounds, r), True,
                 r > 0 and bool((b[1] == 0).any().item())) for r, b in enumerate(blocks)]
    dss = [dist.setup_device(b[0], b[1], b[2], n, bounds, C, sigma, r, world, dev,
                             gathered=gathered) for r, b in enumerate(blocks)]
    rpt, col, val = generate.hamiltonian_device(n)
    full = sb.crs_to_sell_device(rpt, col, val, n, n, C, sigma)
    for x0 in (None, np.inf):
        x = generate.rhs(n)
        if x0 is not None:
            x[0] = x0
        ys = loopback_step(dss, x)
        yf = sb.spmv_sell(full, x)
        for r, y in enumerate(ys):
            r0, r1 = int(bounds[r]), int(bounds[r + 1])
            if x0 is None:
                assert y[: r1 - r0].tobytes() == yf[r0:r1].tobytes(), r
            else:
                np.testing.assert_array_equal(y[: r1 - r0], yf[r0:r1])
    assert all(len(ds.boundary) > 0 and len(ds.interior) > 0 for ds in dss)
