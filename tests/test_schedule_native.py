"""The balanced persistent schedule's work-list arithmetic (csrc/common.cuh), checked on the host:
the real header compiled by nvcc into a small host program (tests/native/balance_check.cu)."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not available")
def test_balanced_schedule_properties(tmp_path):
    exe = tmp_path / "balance_check"
    src = os.path.join(ROOT, "tests", "native", "balance_check.cu")
    subprocess.run(["nvcc", "-std=c++17", "-O1", "-Wno-deprecated-gpu-targets", "-o", str(exe), src], check=True, cwd=ROOT,
                   capture_output=True, timeout=300)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=300)
    assert out.returncode == 0, out.stdout + out.stderr
    assert "configurations OK" in out.stdout
