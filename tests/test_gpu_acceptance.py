"""acceptance.cpp:39-64 on the GPU: EVERY schedule the reference's search
enumerates for every golden family (Adam, MP, PP, and the authored
Reduce/Broadcast program) executes on B200 within 1e-5 of the reference
oracle - coconet::gpu_tune verifies each candidate and raises
CandidateFailed otherwise - and the candidate list and simulated costs are
the reference's own (coconet-ccopt tune --backend sim)."""
import json

import pytest

from tests.cli_util import CLI, cli, dims_args
from tests.dp_util import golden

pytestmark = pytest.mark.gpu

CASES = ["adam_W2_N4096", "adam_W4_N4096", "adam_W8_N65536", "mp_W2_B2_S8_H64", "mp_W4_B2_S8_H64",
         "pp_W2_N4096", "pp_W4_N1024", "rooted_max_W4_N4096"]


@pytest.mark.parametrize("case", CASES)
def test_every_enumerated_schedule_matches_the_oracle_on_gpu(case, tmp_path):
    from paper_2105_05720_b200 import engine
    try:
        engine.load()
    except ImportError:
        pytest.skip("libcoconet_engine.so not built")
    rec = golden(case)
    dims = {k: v for k, v in rec["dims"].items()}
    rep = engine.gpu_tune(rec["base_program"], dims=dims, seed=rec["seed"], reps=1)
    assert len(rep["candidates"]) >= 1
    for c in rep["candidates"]:
        assert c["deviation"] <= 1e-5, c
    if CLI.exists():
        f = tmp_path / "p.json"
        f.write_text(json.dumps(rec["base_program"]))
        ref = json.loads(cli("tune", f, *dims_args(rec), "--backend", "sim", check_rc=0).stdout)
        assert [c["schedule"] for c in rep["candidates"]] == [c["schedule"] for c in ref["candidates"]]
        for a, b in zip(rep["candidates"], ref["candidates"]):
            assert a["simulated_time"] == pytest.approx(b["simulated_time"], rel=1e-12)
            assert a["kernel_steps"] == b["kernel_steps"] and a["comm_bytes"] == b["comm_bytes"]
        assert rep["simulated_winner"] == ref["winner"]
