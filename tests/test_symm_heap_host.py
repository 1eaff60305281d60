"""The symmetric-heap allocator (paper_2105_05720_b200/csrc/symm_heap.h) is
host logic: compiled stand-alone and run on the CPU (tests/native)."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent


def test_symm_heap_allocator(tmp_path):
    gxx = shutil.which("g++")
    if not gxx:
        pytest.skip("g++ not available")
    exe = tmp_path / "symm_heap_test"
    subprocess.run([gxx, "-std=c++17", "-O2", "-I", str(ROOT / "paper_2105_05720_b200" / "csrc"),
                    str(ROOT / "tests" / "native" / "symm_heap_test.cpp"), "-o", str(exe)], check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.startswith("OK"), out.stdout + out.stderr
