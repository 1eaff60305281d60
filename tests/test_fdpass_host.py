"""Descriptor passing of the cuMem heap (paper_2105_05720_b200/csrc/fdpass.h)
is host logic: compiled stand-alone and run between two CPU processes."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_fd_server_hands_a_descriptor_to_another_process(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not available")
    exe = tmp_path / "fdpass_test"
    subprocess.run([gxx, "-std=c++17", "-O2", "-pthread", "-I", str(ROOT / "paper_2105_05720_b200" / "csrc"),
                    str(ROOT / "tests" / "native" / "fdpass_test.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True, timeout=60)
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr
