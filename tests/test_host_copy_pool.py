"""The host thread pool that stages pageable vectors (csrc/sellb_host.cu)
copies every byte for sizes around its 1 MiB threshold and for part counts
that do not divide the size (a round-2 bug left the last bytes uncopied when
n / parts was not a multiple of the 4 KiB part alignment).  Host-only: built
with nvcc, no GPU needed."""

import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
@pytest.mark.parametrize("threads", ["16", "7", "1"])
def test_parallel_copy_is_complete(tmp_path, threads):
    exe = tmp_path / "copy_pool_check"
    subprocess.check_call(
        ["nvcc", "-O2", "-std=c++17", os.path.join(ROOT, "tests/native/copy_pool_check.cu"),
         os.path.join(ROOT, "tests/native/set_error_stub.cu"),
         os.path.join(ROOT, "paper_1307_6209_b200/csrc/sellb_host.cu"), "-o", str(exe),
         "-lpthread"])
    out = subprocess.run([str(exe)], env=dict(os.environ, SELLB_HOST_THREADS=threads),
                         capture_output=True, text=True, timeout=300)
    assert out.returncode == 0
    assert "mismatch" not in out.stdout and "done" in out.stdout, out.stdout
