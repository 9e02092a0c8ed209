"""bench.py's contract pieces that need no GPU: both arms build the same
config dict, the reference arm runs on the host (oracle/_ref or the C port)
and prints one JSON line, and --gpus N outside torchrun refuses to measure
fewer GPUs than asked."""

import json
import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def test_config_dict_is_workload_identity_only():
    import argparse
    import bench
    a = argparse.Namespace(config="cfg5", n=1 << 20, C=32, sigma=512, dtype="f64", gpus=1)
    c1 = bench.bench_config(a, 1)
    assert set(c1) == {"workload", "matrix", "C", "sigma", "dtype", "n_rows", "parallelism",
                       "l2"}
    assert c1["n_rows"] == 1 << 20 and c1["matrix"] == "cfg5"
    c8 = bench.bench_config(a, 8)
    assert c8["parallelism"].startswith("row-blocks x8")


def test_reference_arm_prints_one_line_with_the_same_config():
    out = subprocess.run([sys.executable, "bench.py", "--impl", "reference", "--rows",
                          str(1 << 18), "--steps", "3", "--warmup", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [ln for ln in out.stdout.splitlines() if ln.strip()]
    assert len(lines) == 1
    rec = json.loads(lines[0])
    import argparse
    import bench
    a = argparse.Namespace(config="cfg5", n=1 << 18, C=32, sigma=512, dtype="f64", gpus=1)
    assert rec["config"] == bench.bench_config(a, 1)
    assert rec["impl"] == "reference" and rec["value"] > 0
    assert rec["e2e"]["h2d_bytes_per_step"] == 0 and rec["cpu_baseline"]["cores"] >= 1


def test_gpus_n_refuses_without_the_gpus():
    import torch
    if torch.cuda.device_count() >= 2:
        pytest.skip("this host has the GPUs")
    env = {k: v for k, v in os.environ.items() if k not in ("WORLD_SIZE", "RANK")}
    out = subprocess.run([sys.executable, "bench.py", "--gpus", "2", "--steps", "3"], cwd=ROOT,
                         capture_output=True, text=True, timeout=300, env=env)
    assert out.returncode != 0
    assert "2 GPUs" in (out.stderr + out.stdout)
