"""Test infrastructure (never on the product path): writes
tests/golden/tune_adam_W4_N4096.json, the REFERENCE's own schedule search
(ccopt::tune, autotune.hpp:285-315, compiled from /root/reference headers into
coconet-ccopt and run with --backend sim) on the adam base program at W=4,
N=4096, seed 1 (the program as the reference's program_to_json printed it,
from tests/golden/adam_cases.json). The GPU tests check that coconet::gpu_tune enumerates the same
candidates with the same simulated costs and verifies each on the device.
Usage: python oracle/make_tune_golden.py"""
import json
import subprocess
import sys
import tempfile
from pathlib import Path

ROOT = Path(__file__).resolve().parent.parent
CLI = ROOT / "paper_2105_05720_b200" / "coconet-ccopt"


def main():
    if not CLI.exists():
        sys.exit("needs a coconet-ccopt built against the reference headers")
    case = next(c for c in json.loads((ROOT / "tests" / "golden" / "adam_cases.json").read_text())
                if c["name"] == "adam_W4_N4096")
    with tempfile.NamedTemporaryFile("w", suffix=".json") as f:
        json.dump(case["base_program"], f)
        f.flush()
        out = subprocess.run([str(CLI), "tune", f.name, "--ranks", "4", "--size", "N=4096", "--backend", "sim"],
                             check=True, capture_output=True, text=True).stdout
    rep = json.loads(out)
    rep["program"] = case["base_program"]
    rep["dims"] = {"W": 4, "N": 4096}
    rep["seed"] = 1
    (ROOT / "tests" / "golden" / "tune_adam_W4_N4096.json").write_text(json.dumps(rep, indent=1))
    print("candidates", len(rep["candidates"]), "winner", rep["winner"])


if __name__ == "__main__":
    main()
