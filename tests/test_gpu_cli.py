"""coconet-ccopt with the CUDA backend on B200: the
`ccopt run` flow reproduces the reference Engine's digests on every golden
family, and `tune` ranks the reference's own candidate schedules by measured
device time after verifying each against the oracle."""
import json

import pytest

from tests.cli_util import GOLD, cli, dims_args, need_cli, program_file

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("case", ["adam_W4_N4096", "adam_W8_N4096", "mp_W8_B2_S16_H128", "mp_W4_B2_S8_H64",
                                  "pp_W8_N4096", "pp_W4_N1024"])
def test_run_cuda_matches_reference_digest(tmp_path, case):
    need_cli()
    from tests.dp_util import golden
    try:
        golden(case)
    except KeyError:
        pytest.skip(f"no fixture {case}")
    f, rec = program_file(tmp_path, case, "sched_program")
    j = json.loads(cli("run", f, *dims_args(rec), "--seed", rec.get("seed", 1), check_rc=0).stdout)
    assert j["backend"] == "cuda" and j["math"] == "exact"
    assert j["digest"] == rec["engine_sched_digest"]
    assert j["deviation"] <= 1e-5 and j["device_ms"] > 0
    assert j["lowering"]


def test_run_cuda_fast_within_tolerance(tmp_path):
    need_cli()
    f, rec = program_file(tmp_path, "adam_W4_N4096", "sched_program")
    j = json.loads(cli("run", f, *dims_args(rec), "--math", "fast", check_rc=0).stdout)
    assert j["math"] == "fast" and j["deviation"] <= 1e-5


def _check_tune(j, ref):
    assert [c["schedule"] for c in j["candidates"]] == [c["schedule"] for c in ref["candidates"]]
    for c, r in zip(j["candidates"], ref["candidates"]):
        assert c["simulated_time"] == pytest.approx(r["simulated_time"], rel=1e-12)
        assert c["comm_bytes"] == r["comm_bytes"] and c["kernel_steps"] == r["kernel_steps"]
        assert c["deviation"] <= 1e-5 and c["device_ms"] > 0
    ms = [c["device_ms"] for c in j["candidates"]]
    assert ms[j["winner"]] == min(ms)
    assert j["simulated_winner"] == ref["winner"]
    assert j["ranked_by"] == "device_ms"


def test_tune_cuda_ranks_reference_candidates_by_device_time(tmp_path):
    need_cli()
    ref = json.loads((GOLD / "tune_adam_W4_N4096.json").read_text())
    f = tmp_path / "adam.json"
    f.write_text(json.dumps(ref["program"]))
    j = json.loads(cli("tune", f, "--ranks", "4", "--size", "N=4096", "--reps", "2", check_rc=0).stdout)
    _check_tune(j, ref)


def test_engine_gpu_tune_python_binding():
    from paper_2105_05720_b200 import engine
    ref = json.loads((GOLD / "tune_adam_W4_N4096.json").read_text())
    try:
        engine.load()
    except ImportError:
        pytest.skip("libcoconet_engine.so not built")
    j = engine.gpu_tune(ref["program"], dims={"W": 4, "N": 4096}, reps=2)
    _check_tune(j, ref)


def test_run_cuda_tensor_files_match_sim(tmp_path):
    """--input / --dump on the CUDA backend: the same tensor-file inputs give
    the reference Engine's digest, and the dumped result files are byte-equal
    to the simulated backend's."""
    need_cli()
    import numpy as np

    from oracle import coconet_oracle as co
    f, rec = program_file(tmp_path, "adam_W4_N4096", "sched_program")
    W, N = rec["dims"]["W"], rec["dims"]["N"]
    for name in ("p", "m"):
        arr = np.asarray(co.gen_decl(1, name, [N], "replicated", 0, W), dtype="<f4")
        arr.tofile(str(tmp_path / name) + ".bin")
        (tmp_path / f"{name}.json").write_text(json.dumps({"name": name, "shape": [N], "elem": "f32"}))
    dumps = {}
    for backend in ("cuda", "sim"):
        out = tmp_path / f"dump_{backend}"
        out.mkdir()
        j = json.loads(cli("run", f, *dims_args(rec), "--backend", backend, "--input", f"p={tmp_path / 'p'}",
                           "--input", f"m={tmp_path / 'm'}", "--dump", out, check_rc=0).stdout)
        assert j["digest"] == rec["engine_sched_digest"], backend
        dumps[backend] = {x.name: x.read_bytes() for x in out.iterdir()}
    assert dumps["cuda"] == dumps["sim"]


@pytest.mark.parametrize("case", ["adam_W4_N4096", "mp_W4_B2_S8_H64", "pp_W4_N1024"])
@pytest.mark.parametrize("math", ["exact", "fast"])
def test_run_cuda_is_deterministic(tmp_path, case, math):
    """acceptance.cpp:380-416 runs the CLI twice and byte-compares the JSON.
    On the GPU everything but the measured device time must repeat exactly,
    in FAST math too (fixed reduction order, no atomics in the data path)."""
    need_cli()
    from tests.dp_util import golden
    try:
        golden(case)
    except KeyError:
        pytest.skip(f"no fixture {case}")
    f, rec = program_file(tmp_path, case, "sched_program")
    outs = []
    for _ in range(2):
        j = json.loads(cli("run", f, *dims_args(rec), "--math", math, check_rc=0).stdout)
        for k in ("device_ms", "device_ms_first"):
            j.pop(k)
        outs.append(json.dumps(j, sort_keys=True))
    assert outs[0] == outs[1]


def test_run_cuda_reps_reports_warm_median(tmp_path):
    """`run --reps R` executes R fresh engines (same digest every time, or
    the CLI fails) and reports the median device time after the first."""
    need_cli()
    f, rec = program_file(tmp_path, "adam_W4_N4096", "sched_program")
    j = json.loads(cli("run", f, *dims_args(rec), "--reps", 3, check_rc=0).stdout)
    assert j["runs"] == 3 and j["device_ms"] > 0 and j["device_ms_first"] > 0
    assert j["digest"] == rec["engine_sched_digest"]
