"""Out-of-bounds detection without compute-sanitizer (closed on this pool,
profiles/r02_sanitizer/): every kernel family runs with x embedded between
NaN guard zones and y between canary zones, on device vectors.  A gather
past either end of x turns a row into NaN (caught by the bitwise oracle
comparison); a store outside y's rows -- or, for a chunk range, outside the
range's rows -- overwrites a canary.  Families: the bulk role (pad-skip /
pad-inclusive, U = 4 / 6 / 8, fp32 / fp64), the short-chunk kernel, the
long-row roles (side table, padded reads, row groups), the fp32 TMA ring,
the packed copy, the CRS row-run kernels, the fused unpermute."""

import os
import subprocess
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu
REPO = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

CHILD = r'''
import sys, numpy as np, torch
sys.path.insert(0, "."); sys.path.insert(0, "tests")
import oracle, paper_1307_6209_b200 as sb
from paper_1307_6209_b200 import CRSMatrix, _lib, generate
from test_gpu_long_rows import long_mix
G = 4096
CANARY = np.float64(-1234.5)
lib = _lib.load()
bad = []

def guarded(n, fill, dt):
    buf = torch.full((n + 2 * G,), float(fill), dtype=dt, device="cuda")
    return buf, buf[G:G + n]

def check_sell(tag, m, C, sigma, dt=np.float64, ranges=True):
    if dt == np.float32:
        m = CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val.astype(np.float32))
    s = sb.crs_to_sell(m, C, sigma, dtype=dt)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    tdt = torch.float32 if dt == np.float32 else torch.float64
    xh = generate.rhs(m.n_cols).astype(dt)
    xb, xd = guarded(m.n_cols, float("nan"), tdt)
    xd.copy_(torch.from_numpy(xh))
    y_ref = oracle.spmv_sell(o, xh)
    st = torch.cuda.current_stream().cuda_stream
    spans = [(0, s.n_chunks)]
    if ranges and s.n_chunks > 4:
        spans += [(1, s.n_chunks // 2), (s.n_chunks // 2, s.n_chunks - 1)]
    for c0, c1 in spans:
        yb, yd = guarded(s.n_rows_padded, CANARY, tdt)
        _lib.check(lib.sellb_spmv(s.handle, xd.data_ptr(), yd.data_ptr(), c0, c1, 0, 0, st))
        torch.cuda.synchronize()
        yall = yb.cpu().numpy()
        y = yall[G:G + s.n_rows_padded]
        r0, r1 = c0 * C, c1 * C
        if y[r0:r1].tobytes() != y_ref[r0:r1].tobytes():
            bad.append((tag, "y", c0, c1))
        if not (np.all(yall[:G + r0] == CANARY) and np.all(yall[G + r1:] == CANARY)):
            bad.append((tag, "canary", c0, c1))
    # fused unpermute into a guarded y[n_rows]
    yb, yd = guarded(m.n_rows, CANARY, tdt)
    _lib.check(lib.sellb_spmv(s.handle, xd.data_ptr(), yd.data_ptr(), 0, s.n_chunks, 0, 1, st))
    torch.cuda.synchronize()
    yall = yb.cpu().numpy()
    if yall[G:G + m.n_rows].tobytes() != y_ref[o.perm].tobytes():
        bad.append((tag, "orig"))
    if not (np.all(yall[:G] == CANARY) and np.all(yall[G + m.n_rows:] == CANARY)):
        bad.append((tag, "orig-canary"))
    s.free()

def check_crs(tag, m, unrolled):
    t = {k: torch.from_numpy(np.ascontiguousarray(v)).cuda()
         for k, v in (("rpt", m.rpt), ("col", m.col), ("val", m.val))}
    xh = generate.rhs(m.n_cols)
    xb, xd = guarded(m.n_cols, float("nan"), torch.float64)
    xd.copy_(torch.from_numpy(xh))
    for r0, r1 in ((0, m.n_rows), (5, m.n_rows - 7)):
        yb, yd = guarded(m.n_rows, CANARY, torch.float64)
        _lib.check(lib.sellb_spmv_crs(t["rpt"].data_ptr(), t["col"].data_ptr(),
                                      t["val"].data_ptr(), 0, xd.data_ptr(), yd.data_ptr(),
                                      r0, r1, 0, unrolled, torch.cuda.current_stream().cuda_stream))
        torch.cuda.synchronize()
        yall = yb.cpu().numpy()
        ref = np.full(m.n_rows, CANARY)
        oracle.spmv_crs_range(m.rpt, m.col, m.val, xh, ref, r0, r1, False, bool(unrolled))
        if yall[G:G + m.n_rows].tobytes() != ref.tobytes():
            bad.append((tag, "crs", r0, r1, unrolled))
        if not (np.all(yall[:G] == CANARY) and np.all(yall[G + m.n_rows:] == CANARY)):
            bad.append((tag, "crs-canary", r0, r1, unrolled))

fam = sys.argv[1]
pl = generate.powerlaw(40_000, seed=3, band=900)
if fam == "bulk":
    for dt in (np.float64, np.float32):
        check_sell("stencil", generate.stencil27(20), 32, 1, dt)
        check_sell("laplace", generate.laplace2d(150), 32, 1, dt)
        check_sell("pl128", pl, 32, 128, dt)
        check_sell("plC8", pl, 8, 64, dt)
        check_sell("plC1", pl, 1, 1, dt, ranges=False)
elif fam == "short":
    n = 50_000
    for w in (1, 2):
        rpt = np.arange(n + 1, dtype=np.int64) * w
        col = (np.arange(n * w) % n).astype(np.int32)
        check_sell(f"short{w}", CRSMatrix(n, n, rpt, col, np.linspace(-1, 1, n * w)), 32, 1)
elif fam == "long":
    m = long_mix(5)
    for sig in (1, 512, m.n_rows):
        check_sell(f"long{sig}", m, 32, sig)
    check_sell("longC8", m, 8, m.n_rows)
elif fam == "packed":
    check_sell("packed1", pl, 32, 1)
    check_sell("packedlong", long_mix(5), 32, 1)
elif fam == "crs":
    check_crs("pl", pl, 0)
    check_crs("pl", pl, 1)
    check_crs("long", long_mix(5), 0)
    check_crs("long", long_mix(5), 1)
print("BAD", bad[:10])
print("ok" if not bad else "fail")
'''

CASES = [("bulk", {}), ("bulk", {"SELLB_U": "8"}), ("bulk", {"SELLB_U": "4", "SELLB_VX": "0"}),
         ("bulk", {"SELLB_TMA": "1"}), ("short", {}), ("long", {}),
         ("long", {"SELLB_LONG_SIDE": "0"}), ("long", {"SELLB_LONG_GRP": "1"}),
         ("packed", {"SELLB_PACKED": "1"}), ("crs", {})]


@pytest.mark.parametrize("fam,env", CASES,
                         ids=[f + "-" + ",".join(f"{k[6:]}={v}" for k, v in e.items())
                              for f, e in CASES])
def test_guard_zones(fam, env):
    out = subprocess.run([sys.executable, "-c", CHILD, fam], env=dict(os.environ, **env),
                         capture_output=True, text=True, cwd=REPO, timeout=900)
    assert out.returncode == 0 and out.stdout.strip().endswith("ok"), \
        (out.stdout[-3000:], out.stderr[-3000:])
