"""The tag classifier the kernels use (csrc/common.cuh classify16/classify16b:
bit tricks with one multiply per 8 bytes), compiled for the HOST and checked
against the per-byte definition (R2) on 4M random 16-byte groups,
including every byte value at every position."""
import os
import shutil
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.skipif(shutil.which("nvcc") is None, reason="nvcc not on PATH")
def test_classify16_host(tmp_path):
    exe = tmp_path / "classify16"
    subprocess.run(["nvcc", "-std=c++17", "-O2", "-I", os.path.join(ROOT, "paper_2205_11659_b200", "csrc"),
                    "-o", str(exe), os.path.join(ROOT, "tests", "host", "classify16.cu")], check=True)
    r = subprocess.run([str(exe)], capture_output=True, text=True)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 bad" in r.stdout
