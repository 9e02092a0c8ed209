"""The N>1 leg of bench.py (bench_dist.py) launched the way the driver
launches it -- torchrun, NCCL, one process per GPU -- at world size 1 on the
one GPU this box has (SELLB_FORCE_DIST routes world 1 through the same code).
Checks the stdout contract: exactly one JSON line, even though NCCL prints
its version banner on fd 1 at communicator creation."""

import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


@pytest.mark.parametrize("extra,graph", [
    (["--config", "cfg5", "--rows", str(1 << 21)], "0"),
    (["--config", "cfg5", "--rows", str(1 << 21)], "1"),
    (["--config", "cfg2"], "0")], ids=["cfg5_small", "cfg5_small_graph", "cfg2"])
def test_bench_dist_one_rank_stdout_is_one_json_line(extra, graph):
    env = dict(os.environ, SELLB_FORCE_DIST="1", SELLB_DIST_GRAPH=graph)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "bench.py", "--gpus", "1", "--steps", "20", "--warmup", "3"] + extra
    out = subprocess.run(cmd, env=env, capture_output=True, text=True, cwd=ROOT, timeout=600)
    assert out.returncode == 0, out.stderr[-3000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1, out.stdout
    rec = json.loads(lines[0])
    assert rec["n_gpus"] == 1 and rec["steps"] == 20 and rec["warmup"] == 3
    assert rec["details"]["parity_vs_oracle_all_ranks"] is True
    assert rec["value"] > 0 and rec["gpu_launches"] >= 20
    assert rec["config"]["parallelism"] == "1 GPU"
    assert rec["details"]["step_graph"] is (graph == "1")
    for k in ("exchange_ms", "interior_ms", "boundary_ms", "halo_bytes_per_rank_max"):
        assert k in rec["halo"]


def test_bench_both_arms_print_the_same_config():
    """The driver compares the two arms' config dicts: they must be equal
    (the reference arm's cfg5 block is named in cpu_baseline.sample)."""
    base = [sys.executable, "bench.py", "--steps", "3", "--warmup", "3", "--rows",
            str(1 << 20), "--cpu-budget", "1"]
    recs = []
    for impl in ("ours", "reference"):
        out = subprocess.run(base + ["--impl", impl], capture_output=True, text=True, cwd=ROOT,
                             timeout=900)
        assert out.returncode == 0, out.stderr[-3000:]
        lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
        assert len(lines) == 1, out.stdout
        recs.append(json.loads(lines[0]))
    ours, ref = recs
    assert ours["config"] == ref["config"]
    assert ours["metric"] == ref["metric"] and ours["unit"] == ref["unit"]
    assert ours["details"]["parity_vs_oracle"] is True
    assert ours["e2e"]["matches_device"] is True
    assert ref["impl"] == "reference" and "rows [0, " in ref["cpu_baseline"]["sample"]


def test_nccl_p2p_exchange_replays_from_a_cuda_graph():
    """The mechanics DistSpmv.capture relies on: batch_isend_irecv + wait +
    a consumer kernel captured once, replayed with new data."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "tools/p2p_graph_probe.py"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0 and "graph p2p ok" in out.stdout, out.stderr[-3000:]


def test_dist_step_graph_with_nccl_self_exchange():
    """DistSpmv.capture with NCCL P2P kernels inside the graph (self
    send/recv of a scattered halo through gather/scatter): replay equals the
    eager step bitwise and follows a new x; teardown after release()."""
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1",
           "--master-addr", "127.0.0.1", "--master-port", str(_free_port()),
           "tools/dist_graph_selftest.py"]
    out = subprocess.run(cmd, capture_output=True, text=True, cwd=ROOT, timeout=300)
    assert out.returncode == 0 and "dist graph selftest ok" in out.stdout, out.stderr[-3000:]
