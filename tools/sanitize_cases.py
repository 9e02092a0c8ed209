"""Small instances of every kernel family, each checked against the oracle,
for compute-sanitizer (memcheck / racecheck / synccheck / initcheck):

    compute-sanitizer --tool racecheck python tools/sanitize_cases.py [family]

Families: bulk (pad-skip / pad-incl, fp64 / fp32, U = 4 / 6 / 8), short
(k_spmv_sell_short), long (fused warp-per-row role with and without the side
table, the row-group kernel with named barriers and cp.async rings), tma
(fp32 bulk-copy ring on mbarriers), packed (stored-order copy through the
row-run kernel), crs (row-run kernel), build (device crs_to_sell incl. CUB
sorts / scans), coo, host (pageable-vector staging).
The launch switches are environment variables read once per process, so
each mode of a family runs in its own child process."""

import os
import subprocess
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                "tests"))


def check(m, C, sigma, dtype=np.float64, x0=None, ranges=False):
    import oracle
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import CRSMatrix, generate
    if dtype == np.float32:
        m = CRSMatrix(m.n_rows, m.n_cols, m.rpt, m.col, m.val.astype(np.float32))
    s = sb.crs_to_sell(m, C, sigma, dtype=dtype)
    o = oracle.crs_to_sell(m.rpt, m.col, m.val, m.n_rows, m.n_cols, C, sigma)
    x = generate.rhs(m.n_cols).astype(dtype)
    if x0 is not None:
        x[0] = x0
    y = sb.spmv_sell(s, x)
    with np.errstate(invalid="ignore"):
        yr = oracle.spmv_sell(o, x)
    ok = np.array_equal(y, yr, equal_nan=True) if x0 is not None else y.tobytes() == yr.tobytes()
    ya = sb.spmv_sell(s, x, y=np.ones(s.n_rows_padded, dtype), accumulate=True)
    yo = sb.spmv_sell(s, x, out_order="original")
    ok = ok and np.isfinite(ya).sum() == np.isfinite(yr).sum() and len(yo) == m.n_rows
    for k in ("cs", "cl", "col", "val", "perm", "row_lengths"):
        ok = ok and getattr(s, k).tobytes() == getattr(o, k).tobytes()
    return ok, s


def family(name):
    import paper_1307_6209_b200 as sb
    from paper_1307_6209_b200 import generate
    from test_gpu_long_rows import long_mix
    res = []
    if name == "bulk":
        for dt in (np.float64, np.float32):
            res.append(check(generate.stencil27(24), 32, 1, dt)[0])
            res.append(check(generate.laplace2d(200), 32, 1, dt)[0])
            res.append(check(generate.powerlaw(30_000, seed=3, band=800), 32, 128, dt)[0])
            res.append(check(generate.powerlaw(30_000, seed=3, band=800), 8, 64, dt)[0])
        res.append(check(generate.powerlaw(30_000, seed=3, band=800), 32, 1, x0=np.inf)[0])
    elif name == "short":
        from paper_1307_6209_b200 import CRSMatrix
        n = 100_000
        for w in (1, 2):
            rpt = np.arange(n + 1, dtype=np.int64) * w
            col = (np.arange(n * w) % n).astype(np.int32)
            res.append(check(CRSMatrix(n, n, rpt, col, np.linspace(-1, 1, n * w)), 32, 1)[0])
    elif name == "long":
        m = long_mix(5)
        for sig in (1, 512, 10 ** 9):
            res.append(check(m, 32, sig)[0])
            res.append(check(m, 8, sig if sig < 10 ** 9 else sig)[0])
        res.append(check(m, 32, 10 ** 9, np.float32)[0])
    elif name == "tma":
        res.append(check(generate.stencil27(24), 32, 1, np.float32)[0])
    elif name == "packed":
        for sig in (1, 128):
            ok, s = check(generate.powerlaw(30_000, seed=3, band=800), 32, sig)
            res.append(ok and s.packed)
        res.append(check(long_mix(5), 32, 1)[0])
    elif name == "crs":
        import oracle
        m = generate.powerlaw(30_000, seed=3, band=800)
        x = generate.rhs(m.n_cols)
        for fn, unr in ((sb.spmv_crs, False), (sb.spmv_crs_unrolled, True)):
            ref = oracle.spmv_crs(m.rpt, m.col, m.val, x, m.n_rows, unrolled=unr)
            res.append(fn(m, x).tobytes() == ref.tobytes())
    elif name == "build":
        res.append(check(generate.powerlaw(50_000, seed=7, band=900), 16, 256)[0])
        res.append(check(sb.coo_to_crs(sb.gen_skewed(20_000, 8, 300, 40)), 32, 10 ** 9)[0])
    elif name == "coo":
        rng = np.random.default_rng(1)
        r = rng.integers(0, 3000, 40_000)
        c = rng.integers(0, 2000, 40_000)
        v = rng.uniform(-1, 1, 40_000)
        a = sb.coo_to_crs(sb.COOMatrix(3000, 2000, r, c, v), device=0)
        b = sb.coo_to_crs(sb.COOMatrix(3000, 2000, r, c, v))
        res.append(a.rpt.tobytes() == b.rpt.tobytes() and a.val.tobytes() == b.val.tobytes())
    elif name == "host":
        from paper_1307_6209_b200 import CRSMatrix
        n = 1 << 21
        rp, cl_, vl = generate.hamiltonian_rows(n, 0, n)
        s = sb.crs_to_sell(CRSMatrix(n, n, rp, cl_, vl), 32, 512)
        x = generate.rhs(n)
        y = np.empty(s.n_rows_padded)
        outs = [sb.spmv_sell(s, x, y).copy() for _ in range(3)]
        res.append(all(o.tobytes() == outs[0].tobytes() for o in outs))
    return res


MODES = {
    "bulk": [{}, {"SELLB_U": "4"}, {"SELLB_U": "8"}, {"SELLB_VX": "0"}],
    "short": [{}, {"SELLB_SHORT": "0"}],
    "long": [{}, {"SELLB_LONG_SIDE": "0"}, {"SELLB_LONG_GRP": "1"},
             {"SELLB_LONG_GRP": "1", "SELLB_LONG_MODE": "1"}],
    "tma": [{"SELLB_TMA": "1"}],
    "packed": [{"SELLB_PACKED": "1"}],
    "crs": [{}], "build": [{}], "coo": [{}], "host": [{}],
}

if __name__ == "__main__":
    fams = sys.argv[1:] or list(MODES)
    if os.environ.get("SANITIZE_CHILD"):
        res = family(fams[0])
        print(fams[0], "ok" if all(res) else f"FAILED {res}", flush=True)
        sys.exit(0 if all(res) else 1)
    bad = 0
    for f in fams:
        for env in MODES[f]:
            e = dict(os.environ, SANITIZE_CHILD="1", **env)
            r = subprocess.run([sys.executable, __file__, f], env=e)
            print(f"[{f} {env}] rc={r.returncode}", flush=True)
            bad += r.returncode != 0
    sys.exit(1 if bad else 0)
