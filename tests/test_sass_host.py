"""The built library really contains the Blackwell-native instructions the
design relies on (CPU: cuobjdump over libcoconet_cuda.so, no GPU needed):
tcgen05 MMAs / TMEM loads / TMA for the GEMMs and the LAMB rings, and the
NVSwitch multicast reduction (multimem.ld_reduce -> LDGMC) of the NVLS
kernels, which this round's one-GPU boxes cannot execute."""
import shutil
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
LIB = ROOT / "paper_2105_05720_b200" / "libcoconet_cuda.so"


@pytest.fixture(scope="module")
def sass():
    tool = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not LIB.exists() or not Path(tool).exists():
        pytest.skip("library or cuobjdump missing")
    out = subprocess.run([tool, "-sass", str(LIB)], capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stderr[:500]
    return out.stdout


@pytest.mark.parametrize("mnemonic", ["UTCHMMA", "LDTM", "STTM", "UTMALDG", "UTMASTG", "UBLKCP", "LDGMC"])
def test_sass_contains(sass, mnemonic):
    assert mnemonic in sass, f"{mnemonic} not found in the sm_100a SASS of {LIB.name}"


def test_sass_is_sm100a(sass):
    assert "sm_100a" in sass
