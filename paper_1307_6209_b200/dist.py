"""Row-partitioned multi-GPU SELL-C-sigma SpMV with a halo exchange of x
(SURVEY.md §8(e)); the reference has no distributed mode.

Layout: rank k owns the contiguous rows [b_k, b_{k+1}) (boundaries are
multiples of lcm(C, sigma_eff), balanced by nnz) and the matching slice of
x.  Each rank builds its block's SELL-C-sigma on its own GPU with *global*
column indices -- by the block-decomposition property the
arrays equal the corresponding slice of the single-GPU build -- and keeps a
full-length replica ``x_full`` whose owned part is written locally and whose
halo entries arrive from the owners.

One SpMV (``DistSpmv.step``):
  1. post the halo exchange (NCCL send/recv of the needed x entries, one
     grouped batch; contiguous halos go straight from/into x_full slices,
     scattered ones through gather/scatter kernels),
  2. run the *interior* chunks (every column owned) while it is in flight,
  3. wait, unpack, run the *boundary* chunks,
  4. apply the padding fix-up with rank 0's x[0] (the reference adds
     0*x[0] per padded slot; only a non-finite x[0] changes y).
Every row is summed by one thread in slot order, so y is bitwise identical
to the single-GPU product and to the reference.

The communication and partition logic is backend-agnostic: on GPUs it runs
over NCCL with the CUDA kernels (``CudaEngine``); the CPU tests drive the
same code over gloo with a checker engine built on the oracle.
"""

import math
import os
import sys

import numpy as np

from .errors import ParameterError

try:
    import torch
    import torch.distributed as tdist
except ImportError:  # pragma: no cover
    torch = None
    tdist = None


# ---------------------------------------------------------------------------
# partition
# ---------------------------------------------------------------------------

def sigma_effective(n_rows, C, sigma):
    """formats.py:325-334 (None when sigma >= n: one global scope)."""
    if sigma <= C:
        return 1
    if sigma >= n_rows:
        return None
    if sigma % C:
        raise ParameterError(
            f"sigma ({sigma}) must be a multiple of C ({C}) when C < sigma < n_rows")
    return sigma


def partition_rows(rpt, world, C=32, sigma=1):
    """Contiguous row blocks for ``world`` ranks, boundaries at multiples of
    lcm(C, sigma_eff), balanced by nonzeros.  Returns int64 bounds[world+1].

    A global scope (sigma >= n_rows) does not decompose; it is rejected for
    world > 1 (sort per block with sigma <= rows per rank instead)."""
    rpt = np.asarray(rpt, dtype=np.int64)
    n = len(rpt) - 1
    s_eff = sigma_effective(n, C, sigma)
    if s_eff is None:
        if world > 1:
            raise ParameterError("sigma >= n_rows (global sort) cannot be row-partitioned")
        s_eff = 1
    unit = C * s_eff // math.gcd(C, s_eff)
    nnz = int(rpt[-1])
    bounds = [0]
    for k in range(1, world):
        target = nnz * k / world
        r = int(np.searchsorted(rpt, target, side="left"))
        r = int(round(r / unit)) * unit
        r = min(max(r, bounds[-1]), n)
        bounds.append(r)
    bounds.append(n)
    return np.array(bounds, dtype=np.int64)


# ---------------------------------------------------------------------------
# halo plan
# ---------------------------------------------------------------------------

def _contiguous(idx):
    return len(idx) > 0 and int(idx[-1]) - int(idx[0]) + 1 == len(idx)


class HaloPlan:
    """Who sends which x entries to whom.

    ``recv[p]``: sorted global indices this rank needs from rank p;
    ``send[p]``: sorted global indices (owned here) rank p needs from us.
    Built with one all_gather of the request lists (setup only).

    x[0] is never part of a halo: rank 0 sends it on its own to every rank
    that reads it (a real column-0 entry, or the reference's 0*x[0] padding
    term), into a separate one-element buffer, so no receive ever writes
    x_full[0] while the interior chunks may read it (DistSpmv.step)."""

    def __init__(self, rank, world, bounds, recv, send, need_x0):
        self.rank, self.world = rank, world
        self.bounds = np.asarray(bounds, dtype=np.int64)
        self.recv = recv
        self.send = send
        self.need_x0 = need_x0          # rank -> bool: that rank needs x[0]

    @staticmethod
    def requests(col_local, bounds, rank):
        """The x entries this rank's block reads but does not own, by owner."""
        bounds = np.asarray(bounds, dtype=np.int64)
        r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
        col = np.asarray(col_local)
        remote = np.unique(col[(col < r0) | (col >= r1)]).astype(np.int64)
        remote = remote[remote != 0]                 # x[0] travels separately
        owner = np.searchsorted(bounds, remote, side="right") - 1
        return {int(p): remote[owner == p].astype(np.int32)
                for p in np.unique(owner) if p != rank}

    @staticmethod
    def reads_x0(col_local, bounds, rank):
        """Whether this rank's block has a real entry in (non-owned) column 0."""
        return rank != 0 and int(bounds[rank]) > 0 and bool(np.any(np.asarray(col_local) == 0))

    @classmethod
    def from_requests(cls, rank, world, bounds, gathered):
        """gathered[p] = (requests of rank p, rank p has padding[, rank p reads
        column 0 as a real entry])."""
        recv = gathered[rank][0]
        send = {}
        for p in range(world):
            if p == rank:
                continue
            want = gathered[p][0].get(rank)
            if want is not None and len(want):
                send[p] = np.asarray(want, dtype=np.int32)
        need_x0 = {p: p != 0 and (bool(gathered[p][1]) or
                                  (len(gathered[p]) > 2 and bool(gathered[p][2])))
                   for p in range(world)}
        return cls(rank, world, bounds, recv, send, need_x0)

    @classmethod
    def build(cls, col_local, bounds, rank, world, has_padding, group=None):
        recv = cls.requests(col_local, bounds, rank)
        gathered = [None] * world
        tdist.all_gather_object(gathered, (recv, bool(has_padding),
                                           cls.reads_x0(col_local, bounds, rank)), group=group)
        return cls.from_requests(rank, world, bounds, gathered)

    def halo_entries(self):
        return int(sum(len(v) for v in self.recv.values()))

    def bytes_per_step(self, value_bytes=8):
        """Bytes this rank receives per SpMV (x halo + x[0])."""
        return value_bytes * (self.halo_entries() + (1 if self.need_x0.get(self.rank) else 0))


def classify_chunks(rpt_local, col_local, perm, C, r0, r1):
    """Boundary flag per chunk: a stored row with a non-owned column makes
    its chunk wait for the halo.  Returns (interior_ranges, boundary_ranges)
    as lists of [c0, c1) runs."""
    rpt_local = np.asarray(rpt_local, dtype=np.int64)
    n = len(rpt_local) - 1
    col = np.asarray(col_local)
    remote = ((col < r0) | (col >= r1)).astype(np.int64)
    cnt = np.zeros(len(remote) + 1, dtype=np.int64)
    np.cumsum(remote, out=cnt[1:])
    per_row = (cnt[rpt_local[1:]] - cnt[rpt_local[:-1]]) > 0
    n_chunks = (n + C - 1) // C
    bnd = np.zeros(n_chunks, dtype=bool)
    if n:
        np.logical_or.at(bnd, np.asarray(perm, dtype=np.int64)[per_row] // C, True)
    return _runs(~bnd), _runs(bnd)


def _runs(mask):
    runs = []
    i, n = 0, len(mask)
    while i < n:
        if mask[i]:
            j = i
            while j < n and mask[j]:
                j += 1
            runs.append((i, j))
            i = j
        else:
            i += 1
    return runs


# ---------------------------------------------------------------------------
# engines: the local multiply
# ---------------------------------------------------------------------------

class CudaEngine:
    """Local SELL multiply on this rank's GPU through libsellb200.so."""

    def __init__(self, sell, device):
        from . import _lib
        self.lib = _lib.load()
        self.check = _lib.check
        self.sell = sell
        self.handle = sell.handle
        self.device = device
        self.dtype_code = _lib.SELLB_F32 if sell.dtype == np.float32 else _lib.SELLB_F64
        self.launches = 0

    def stream(self):
        return torch.cuda.current_stream(self.device).cuda_stream

    def run_ranges(self, ranges, x_full, y):
        st = self.stream()
        for c0, c1 in ranges:
            self.check(self.lib.sellb_spmv(self.handle, x_full.data_ptr(), y.data_ptr(),
                                           c0, c1, 0, 0, st))
            self.launches += 1

    def gather(self, x_full, idx_dev, out):
        self.check(self.lib.sellb_gather(x_full.data_ptr(), idx_dev.data_ptr(),
                                         out.data_ptr(), idx_dev.numel(), self.dtype_code,
                                         self.stream()))
        self.launches += 1

    def scatter(self, buf, idx_dev, x_full):
        self.check(self.lib.sellb_scatter(buf.data_ptr(), idx_dev.data_ptr(),
                                          x_full.data_ptr(), idx_dev.numel(), self.dtype_code,
                                          self.stream()))
        self.launches += 1

    def pad_fixup(self, x0_buf, y):
        self.check(self.lib.sellb_pad_fixup(self.handle, x0_buf.data_ptr(), y.data_ptr(),
                                            self.stream()))
        self.launches += 1


# ---------------------------------------------------------------------------
# the distributed SpMV
# ---------------------------------------------------------------------------

class DistSpmv:
    """One rank's share of y = A x.

    ``engine`` runs local chunk ranges (CudaEngine on GPUs); ``sell_host``
    supplies n_chunks / row info; x_full / y are torch tensors on the
    engine's device (CPU tensors under gloo)."""

    def __init__(self, engine, plan, n_chunks, n_pad, n_global, interior, boundary,
                 has_padding, device, dtype, group=None):
        self.engine, self.plan = engine, plan
        self.interior, self.boundary = interior, boundary
        self.group = group
        self.device = device
        r0, r1 = int(plan.bounds[plan.rank]), int(plan.bounds[plan.rank + 1])
        self.r0, self.r1 = r0, r1
        self.x_full = torch.zeros(n_global, dtype=dtype, device=device)
        self.x_local = self.x_full[r0:r1]               # owned slice (a view)
        self.y = torch.zeros(n_pad, dtype=dtype, device=device)
        self.has_padding = has_padding
        self.x0_buf = torch.zeros(1, dtype=dtype, device=device)
        idx = lambda a: torch.from_numpy(np.ascontiguousarray(a, dtype=np.int32)).to(device)
        # receive side: contiguous halos land directly in x_full
        self.recv_ops = []
        for p, g in sorted(plan.recv.items()):
            if _contiguous(g):
                self.recv_ops.append((p, self.x_full[int(g[0]):int(g[-1]) + 1], None))
            else:
                self.recv_ops.append((p, torch.empty(len(g), dtype=dtype, device=device),
                                      idx(g)))
        self.send_ops = []
        for p, g in sorted(plan.send.items()):
            if _contiguous(g):
                self.send_ops.append((p, self.x_full[int(g[0]):int(g[-1]) + 1], None))
            else:
                self.send_ops.append((p, torch.empty(len(g), dtype=dtype, device=device),
                                      idx(g)))
        self.x0_peers = [p for p, need in plan.need_x0.items() if need] \
            if plan.rank == 0 else []
        self.x0_recv = plan.need_x0.get(plan.rank, False)

    def _post_exchange(self):
        ops = []
        for p, buf, gidx in self.send_ops:
            if gidx is not None:
                self.engine.gather(self.x_full, gidx, buf)
            ops.append(tdist.P2POp(tdist.isend, buf, p, group=self.group))
        for p, buf, _ in self.recv_ops:
            ops.append(tdist.P2POp(tdist.irecv, buf, p, group=self.group))
        for p in self.x0_peers:
            ops.append(tdist.P2POp(tdist.isend, self.x_full[0:1], p, group=self.group))
        if self.x0_recv:
            ops.append(tdist.P2POp(tdist.irecv, self.x0_buf, 0, group=self.group))
        return tdist.batch_isend_irecv(ops) if ops else []

    graph = None
    graph_launches = 0      # library kernels recorded in the graph (one step)

    def step(self):
        """y_local = A_local x (x_local must hold this rank's x slice)."""
        if self.graph is not None:
            self.graph.replay()
            return self.y
        return self._step_eager()

    def capture(self):
        """Record one step -- exchange post, interior, wait, boundary, x[0]
        fix-up -- in a CUDA graph so later steps cost one replay of host
        time instead of ~40-90 us of NCCL post per step
        (profiles/r01f_p2p_overhead.txt).  Collective: every rank must call
        it.  The graph is kept only if its replay -- with every halo entry,
        receive buffer and x[0] poisoned with NaN beforehand -- reproduces the
        eager y bitwise on EVERY rank (MIN-reduced flag); otherwise all ranks
        stay eager.  Returns whether the graph is in use.

        Known limit: if the capture fails on one rank after its P2P batch was
        recorded and not on another, the ranks' NCCL P2P sequences may no
        longer match and the eager fallback step can hang; the bench leg
        therefore keeps the graph opt-in (SELLB_DIST_GRAPH=1) and the
        multi-rank tests run under a timeout."""
        if self.device.type != "cuda":
            return False
        def all_ok(v):
            flag = torch.tensor([v], dtype=torch.float32, device=self.device)
            tdist.all_reduce(flag, op=tdist.ReduceOp.MIN, group=self.group)
            return float(flag.item()) == 1.0

        def dbg(msg):
            if os.environ.get("SELLB_DIST_DEBUG"):
                print(f"[capture] {msg}", file=sys.stderr, flush=True)

        g, y_ref, ok = None, None, 1.0
        try:
            self._step_eager()              # communicators exist before capture
            torch.cuda.synchronize(self.device)
            y_ref = self.y.clone()
            dbg("eager step done")
            g = torch.cuda.CUDAGraph()
            l0 = self.engine.lib.sellb_launch_count()
            # thread_local: the NCCL watchdog thread may query events meanwhile
            with torch.cuda.graph(g, capture_error_mode="thread_local"):
                self._step_eager()
            self.graph_launches = int(self.engine.lib.sellb_launch_count() - l0)
            dbg(f"captured ({self.graph_launches} library launches)")
        except Exception as e:              # capture unsupported here: stay eager
            dbg(f"capture failed: {e!r}")
            ok = 0.0
        # replay only when EVERY rank captured: a replayed NCCL send/recv whose
        # peer does not replay would wait forever
        if all_ok(ok):
            ok = 1.0
            try:
                self.y.zero_()
                # poison everything the exchange must deliver: a replay whose
                # receives land nothing cannot reproduce y_ref
                self.x_full[:self.r0].fill_(float("nan"))
                self.x_full[self.r1:].fill_(float("nan"))
                self.x0_buf.fill_(float("nan"))
                for _, buf, gidx in self.recv_ops:
                    if gidx is not None:
                        buf.fill_(float("nan"))
                torch.cuda.synchronize(self.device)
                dbg("replaying")
                g.replay()
                torch.cuda.synchronize(self.device)
                dbg("replayed")
                iv = torch.int64 if self.y.element_size() == 8 else torch.int32
                ok = 1.0 if bool(torch.equal(self.y.view(iv), y_ref.view(iv))) else 0.0
            except Exception:
                ok = 0.0
        else:
            ok = 0.0
        flag = torch.tensor([ok], dtype=torch.float32, device=self.device)
        tdist.all_reduce(flag, op=tdist.ReduceOp.MIN, group=self.group)
        self.graph = g if float(flag.item()) == 1.0 else None
        if self.graph is None:
            self._step_eager()              # leave y as an eager step made it
            torch.cuda.synchronize(self.device)
        return self.graph is not None

    def release(self):
        """Drop the step graph.  Call before destroy_process_group(): with
        NCCL kernels captured, the teardown hangs while the graph is alive
        (tools/p2p_graph_probe.py)."""
        if self.graph is not None:
            torch.cuda.synchronize(self.device)
            self.graph = None

    def _nvtx(self, name):
        if self.device.type == "cuda":
            torch.cuda.nvtx.range_push(name)

    def _nvtx_pop(self):
        if self.device.type == "cuda":
            torch.cuda.nvtx.range_pop()

    def _step_eager(self):
        self._nvtx("dist.step")
        if self.x0_recv:
            # the interior chunks may read x_full[0] (padding: 0 * x[0]); it
            # holds +0.0 until the exchange has landed, so a previous step's
            # non-finite x[0] cannot leak into them -- the fix-up below adds
            # 0 * x[0] for the current one
            self.x_full[0:1].zero_()
        works = self._post_exchange()
        self._nvtx("dist.interior")
        self.engine.run_ranges(self.interior, self.x_full, self.y)
        self._nvtx_pop()
        for w in works:
            w.wait()
        if self.x0_recv:
            self.x_full[0:1].copy_(self.x0_buf)
        for p, buf, gidx in self.recv_ops:
            if gidx is not None:
                self.engine.scatter(buf, gidx, self.x_full)
        self._nvtx("dist.boundary")
        self.engine.run_ranges(self.boundary, self.x_full, self.y)
        self._nvtx_pop()
        if self.x0_recv and self.has_padding:
            self.engine.pad_fixup(self.x0_buf, self.y)
        self._nvtx_pop()
        return self.y


def setup(crs_local, bounds, C, sigma, rank, world, device, engine_factory,
          dtype=None, group=None, plan=None, built=None):
    """Build this rank's local SELL (through ``engine_factory(crs_local)``,
    which returns (engine, sell_info)) and the halo plan (collective unless a
    precomputed ``plan`` is given)."""
    engine, info = built if built is not None else engine_factory(crs_local)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    perm = info["perm"]
    has_padding = bool(info["has_padding"])
    if plan is None:
        plan = HaloPlan.build(crs_local.col, bounds, rank, world, has_padding, group=group)
    interior, boundary = classify_chunks(crs_local.rpt, crs_local.col, perm, C, r0, r1)
    tdt = dtype or torch.float64
    return DistSpmv(engine, plan, info["n_chunks"], info["n_rows_padded"],
                    crs_local.n_cols, interior, boundary, has_padding, device, tdt,
                    group=group)


def requests_torch(col_t, bounds, rank):
    """HaloPlan.requests on a (device) torch tensor of local column indices:
    sorted unique non-owned columns grouped by owner, computed where the
    matrix lives (torch.unique / searchsorted on the GPU)."""
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    remote = torch.unique(col_t[(col_t < r0) | (col_t >= r1)])
    remote = remote[remote != 0]                     # x[0] travels separately
    if remote.numel() == 0:
        return {}
    b = torch.as_tensor(np.asarray(bounds, dtype=np.int64), device=col_t.device)
    owner = torch.searchsorted(b, remote.to(torch.int64), right=True) - 1
    out = {}
    for p in torch.unique(owner).tolist():
        if p != rank:
            out[int(p)] = remote[owner == p].to(torch.int32).cpu().numpy()
    return out


def setup_device(rpt_t, col_t, val_t, n_global, bounds, C, sigma, rank, world, device,
                 group=None, gathered=None):
    """Row-partitioned setup for a block whose CRS is already in HBM (torch
    tensors on `device`, global column indices): device build, halo plan and
    interior/boundary split without a host copy of the block (cfg5: ~2 GB
    of CRS per GPU at 8 GPUs).  ``gathered`` replaces the all_gather of the
    request lists (single-process loopback tests)."""
    from . import _lib
    from .formats import crs_to_sell_device
    n_local = rpt_t.numel() - 1
    s = crs_to_sell_device(rpt_t, col_t, val_t, n_local, n_global, C, sigma,
                           device=device.index or 0)
    if world > 1 and s.shadow:
        s.set_shadow(False)     # interior / boundary chunk runs keep the block's own layout
    info = s.info()
    has_padding = info.slots > info.nnz
    if gathered is None:
        plan_req = requests_torch(col_t, bounds, rank)
        reads0 = rank != 0 and int(bounds[rank]) > 0 and bool((col_t == 0).any().item())
        gathered = [None] * world
        tdist.all_gather_object(gathered, (plan_req, bool(has_padding), reads0), group=group)
    plan = HaloPlan.from_requests(rank, world, bounds, gathered)
    r0, r1 = int(bounds[rank]), int(bounds[rank + 1])
    remote = ((col_t < r0) | (col_t >= r1)).to(torch.int64)
    cnt = torch.zeros(remote.numel() + 1, dtype=torch.int64, device=col_t.device)
    torch.cumsum(remote, 0, out=cnt[1:])
    row_flag = ((cnt[rpt_t[1:]] - cnt[rpt_t[:-1]]) > 0).to(torch.uint8).contiguous()
    chunk_flag = torch.empty(info.n_chunks, dtype=torch.uint8, device=col_t.device)
    _lib.check(_lib.load().sellb_chunk_flags(s.handle, row_flag.data_ptr(),
                                             chunk_flag.data_ptr(),
                                             torch.cuda.current_stream(device).cuda_stream))
    bnd = chunk_flag.cpu().numpy().astype(bool)
    del remote, cnt, row_flag
    engine = CudaEngine(s, device)
    tdt = torch.float32 if s.dtype == np.float32 else torch.float64
    return DistSpmv(engine, plan, info.n_chunks, info.n_rows_padded, n_global, _runs(~bnd),
                    _runs(bnd), has_padding, device, tdt, group=group)


def cuda_engine_factory(C, sigma, device, dtype=None):
    """engine_factory for GPUs: device build of the local block."""
    from .formats import crs_to_sell

    def make(crs_local):
        s = crs_to_sell(crs_local, C, sigma, device=device.index or 0, dtype=dtype)
        if s.shadow:
            s.set_shadow(False)  # interior / boundary chunk runs keep the block's own layout
        rl = s.row_lengths
        cl = s.cl
        has_pad = bool(len(rl) and np.any(rl < np.repeat(cl, C)))
        info = {"perm": s.perm, "n_chunks": s.n_chunks, "n_rows_padded": s.n_rows_padded,
                "has_padding": has_pad, "sell": s}
        return CudaEngine(s, device), info
    return make


# ---------------------------------------------------------------------------
# partition helper for the cfg5 strong-scaling layout
# ---------------------------------------------------------------------------

def _cfg5_bounds(n, world, C, sigma):
    """Equal row blocks aligned to lcm(C, sigma_eff) (cfg5 rows carry ~19.7
    entries each, so equal rows balance the nonzeros)."""
    s_eff = sigma_effective(n, C, sigma) or 1
    unit = C * s_eff // math.gcd(C, s_eff)
    b = [min(n, int(round(n * k / world / unit)) * unit) for k in range(world)] + [n]
    return np.array(b, dtype=np.int64)
