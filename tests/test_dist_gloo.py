"""Multi-rank path on CPU: world_size 2 (and 3) over gloo.

The partition, halo plan, exchange, interior/boundary split and padding
fix-up of paper_1307_6209_b200.dist run unchanged; only the local multiply is
the oracle (the checker) instead of the CUDA engine, since this host has no
GPU.  The concatenated y must equal the single-process oracle product
bit for bit, including the NaN rows a non-finite x[0] produces.
"""

import socket

import numpy as np
import pytest
import torch
import torch.distributed as tdist
import torch.multiprocessing as mp

import oracle
from paper_1307_6209_b200 import CRSMatrix, dist, generate


class OracleEngine:
    """Test-only engine: the CPU checker behind the DistSpmv interface."""

    def __init__(self, o):
        self.o = o
        self.launches = 0

    def run_ranges(self, ranges, x_full, y):
        xf, yy = x_full.numpy(), y.numpy()
        for c0, c1 in ranges:
            oracle.spmv_sell_range(self.o.cs, self.o.cl, self.o.C, self.o.col, self.o.val,
                                   xf, yy, c0, c1, False)

    def gather(self, x_full, idx, out):
        out.copy_(x_full[idx.long()])

    def scatter(self, buf, idx, x_full):
        x_full[idx.long()] = buf

    def pad_fixup(self, x0_buf, y):
        x0 = float(x0_buf[0])
        if np.isfinite(x0):
            return
        rl = self.o.row_lengths
        cap = np.repeat(self.o.cl, self.o.C)
        yy = y.numpy()
        with np.errstate(invalid="ignore"):
            yy[rl < cap] = yy[rl < cap] + 0.0 * x0


def oracle_factory(C, sigma):
    def make(crs):
        o = oracle.crs_to_sell(crs.rpt, crs.col, crs.val, crs.n_rows, crs.n_cols, C, sigma)
        has_pad = bool(np.any(o.row_lengths < np.repeat(o.cl, C)))
        return OracleEngine(o), {"perm": o.perm, "n_chunks": o.n_chunks,
                                 "n_rows_padded": o.n_rows_padded, "has_padding": has_pad}
    return make


def banded(n, seed):
    rng = np.random.default_rng(seed)
    offs = np.array([-40, -7, -3, -1, 0, 1, 2, 9, 33])
    rows = np.repeat(np.arange(n), len(offs))
    cols = rows + np.tile(offs, n)
    keep = (cols >= 0) & (cols < n) & ((rng.random(len(cols)) < 0.7) | (cols == rows))
    rows, cols = rows[keep], cols[keep]
    rpt = np.zeros(n + 1, np.int64)
    np.cumsum(np.bincount(rows, minlength=n), out=rpt[1:])
    return CRSMatrix(n, n, rpt, cols, rng.uniform(-1, 1, len(cols)))


def block(m, r0, r1):
    s, e = m.rpt[r0], m.rpt[r1]
    return CRSMatrix(r1 - r0, m.n_cols, m.rpt[r0:r1 + 1] - s, m.col[s:e], m.val[s:e])


def _worker(rank, world, port, case, C, sigma, q):
    try:
        tdist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}",
                                 rank=rank, world_size=world)
        m = case()
        bounds = (dist._cfg5_bounds(m.n_rows, world, C, sigma) if case is case_cfg5
                  else dist.partition_rows(m.rpt, world, C, sigma))
        loc = block(m, int(bounds[rank]), int(bounds[rank + 1]))
        ds = dist.setup(loc, bounds, C, sigma, rank, world, torch.device("cpu"),
                        oracle_factory(C, sigma))
        out = {}
        # the order matters: a finite x[0] right after a non-finite one must
        # not inherit it (x[0] travels apart from the halo)
        for tag, x0 in (("finite", None), ("inf", np.inf), ("finite_after_inf", None),
                        ("nan", np.nan), ("finite_after_nan", None)):
            x = generate.rhs(m.n_cols)
            if x0 is not None:
                x[0] = x0
            ds.x_local.copy_(torch.from_numpy(x[ds.r0:ds.r1]))
            y = ds.step().numpy().copy()
            out[tag] = y
        q.put((rank, out, ds.plan.halo_entries(), len(ds.interior), len(ds.boundary), None))
        tdist.destroy_process_group()
    except Exception as exc:  # surface worker failures in the parent
        import traceback
        q.put((rank, None, 0, 0, 0, traceback.format_exc()))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def run_world(world, case, C, sigma):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, C, sigma, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    for r in res:
        assert r[5] is None, r[5]
    return sorted(res, key=lambda r: r[0])


def case_banded():
    return banded(3001, 4)


def case_stencil():
    return generate.stencil27(12, nz=16)


def case_powerlaw():
    return generate.powerlaw(4000, seed=9, band=300)


def case_arrow():
    """Banded plus real entries in column 0 on every 7th row: ranks other
    than 0 read x[0] as a matrix entry, not only as padding."""
    m = banded(2003, 6)
    rows = np.arange(m.n_rows)
    extra = rows[(rows % 7 == 3)]
    rr = np.concatenate([np.repeat(rows, np.diff(m.rpt)), extra])
    cc = np.concatenate([m.col, np.zeros(len(extra), dtype=m.col.dtype)])
    vv = np.concatenate([m.val, np.full(len(extra), 0.5)])
    key = rr * m.n_cols + cc
    key, first = np.unique(key, return_index=True)
    rr, cc, vv = key // m.n_cols, key % m.n_cols, vv[first]
    rpt = np.zeros(m.n_rows + 1, np.int64)
    np.cumsum(np.bincount(rr, minlength=m.n_rows), out=rpt[1:])
    return CRSMatrix(m.n_rows, m.n_cols, rpt, cc.astype(np.int32), vv)


def case_cfg5():
    """The cfg5 generator's structure (hopping offsets up to +-2^20 scaled
    down: N = 2^16, so the +-4096 / +-65536 hops cross every rank) in the
    strong-scaling layout: _cfg5_bounds, SELL-32-512."""
    return generate.hamiltonian(1 << 16)


def single(m, C, sigma, x):
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    with np.errstate(invalid="ignore"):
        return o, oracle.spmv_sell(o, x)


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("case,C,sigma", [(case_banded, 32, 1), (case_banded, 8, 64),
                                          (case_stencil, 32, 1), (case_powerlaw, 32, 128),
                                          (case_arrow, 32, 1)])
def test_distributed_equals_single(world, case, C, sigma):
    check_world(world, case, C, sigma)


def test_cfg5_layout_world4():
    """World 4 over gloo on the cfg5 strong-scaling layout (oracle engine)."""
    check_world(4, case_cfg5, 32, 512)


def check_world(world, case, C, sigma):
    m = case()
    bounds = (dist._cfg5_bounds(m.n_rows, world, C, sigma) if case is case_cfg5
              else dist.partition_rows(m.rpt, world, C, sigma))
    res = run_world(world, case, C, sigma)
    for tag, x0 in (("finite", None), ("inf", np.inf), ("finite_after_inf", None),
                    ("nan", np.nan), ("finite_after_nan", None)):
        x = generate.rhs(m.n_cols)
        if x0 is not None:
            x[0] = x0
        for rank, out, halo, n_int, n_bnd, _ in res:
            r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
            # block-decomposition: the block's own build equals the global slice
            _, y_ref = single(block(m, r0, r1), C, sigma, x)
            if x0 is None:
                assert out[tag].tobytes() == y_ref.tobytes(), (rank, tag)
            else:
                np.testing.assert_array_equal(out[tag], y_ref)
        # and the stitched result equals the single-GPU product (stored order
        # of each block = global stored order when boundaries are lcm-aligned)
        if x0 is None:
            o_all, y_all = single(m, C, sigma, x)
            stitched = np.concatenate([r[1][tag][: int(bounds[r[0] + 1] - bounds[r[0]])]
                                       for r in res])
            assert stitched.tobytes() == y_all[: m.n_rows].tobytes()
    assert all(r[2] > 0 for r in res)          # every rank has a halo
    assert sum(r[3] for r in res) > 0           # some interior work overlaps


def test_partition_alignment_and_balance():
    m = generate.powerlaw(10000, seed=2, band=500)
    for world in (2, 4, 8):
        b = dist.partition_rows(m.rpt, world, 32, 128)
        assert b[0] == 0 and b[-1] == m.n_rows
        assert all(int(v) % 128 == 0 for v in b[1:-1])
        nnz = np.diff(m.rpt[b])
        assert nnz.max() < 1.3 * m.nnz / world
    with pytest.raises(Exception):
        dist.partition_rows(m.rpt, 2, 32, 10 ** 9)


def test_classify_chunks_banded():
    m = banded(640, 1)
    loc = block(m, 320, 640)
    o = oracle.crs_to_sell(loc.rpt, loc.col, loc.val, loc.n_rows, loc.n_cols, 32, 1)
    interior, boundary = dist.classify_chunks(loc.rpt, loc.col, o.perm, 32, 320, 640)
    assert boundary[0][0] == 0                  # first rows reach below row 320
    covered = sorted(interior + boundary)
    assert covered[0][0] == 0 and covered[-1][1] == o.n_chunks
