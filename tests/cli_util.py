"""Helpers for the coconet-ccopt CLI tests (the reference CLI flow with a
CUDA backend, paper_2105_05720_b200/csrc/cli/coconet_ccopt.cpp)."""
import json
import subprocess
from pathlib import Path

import pytest

from tests.dp_util import golden

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2105_05720_b200" / "coconet-ccopt"
GOLD = ROOT / "tests" / "golden"


def need_cli():
    if not CLI.exists():
        pytest.skip("coconet-ccopt is built only where the reference DSL headers exist")


def program_file(tmp_path, case: str, which: str) -> tuple[Path, dict]:
    rec = golden(case)
    f = tmp_path / f"{case}_{which}.json"
    f.write_text(json.dumps(rec[which]))
    return f, rec


def cli(*args, check_rc=None):
    p = subprocess.run([str(CLI)] + [str(a) for a in args], capture_output=True, text=True, timeout=600)
    if check_rc is not None:
        assert p.returncode == check_rc, (p.returncode, p.stderr[-2000:])
    return p


def dims_args(rec):
    d = rec["dims"]
    out = ["--ranks", str(d["W"])]
    for k, v in d.items():
        if k != "W":
            out += ["--size", f"{k}={v}"]
    return out
