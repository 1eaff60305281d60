"""coconet-ccopt on the host (no GPU): the reference CLI contract — the
subcommands that never touch the data path, the simulated backend reproducing
the reference Engine's golden digests, argument errors (exit 2), and that the
CUDA backend fails loudly without a device instead of falling back."""
import json

from tests.cli_util import GOLD, cli, dims_args, need_cli, program_file


def test_check_and_transform(tmp_path):
    need_cli()
    f, rec = program_file(tmp_path, "adam_W4_N4096", "base_program")
    j = json.loads(cli("check", f, *dims_args(rec), check_rc=0).stdout)
    assert j["world_size"] == 4 and j["diagnostics"] == []
    assert any(n["kind"] == "allreduce" for n in j["nodes"])


def test_run_sim_reproduces_reference_digests(tmp_path):
    need_cli()
    for case in ("adam_W4_N4096", "adam_W2_N1024"):
        f, rec = program_file(tmp_path, case, "sched_program")
        j = json.loads(cli("run", f, *dims_args(rec), "--backend", "sim", check_rc=0).stdout)
        assert j["digest"] == rec["engine_sched_digest"]
        assert j["backend"] == "sim" and j["deviation"] <= 1e-5


def test_tune_sim_matches_committed_reference_search(tmp_path):
    need_cli()
    ref = json.loads((GOLD / "tune_adam_W4_N4096.json").read_text())
    f = tmp_path / "adam.json"
    f.write_text(json.dumps(ref["program"]))
    j = json.loads(cli("tune", f, "--ranks", "4", "--size", "N=4096", "--backend", "sim", check_rc=0).stdout)
    assert [c["schedule"] for c in j["candidates"]] == [c["schedule"] for c in ref["candidates"]]
    assert j["winner"] == ref["winner"]


def test_argument_errors_exit_2(tmp_path):
    need_cli()
    f, rec = program_file(tmp_path, "adam_W4_N4096", "base_program")
    assert cli("run", f, "--bogus").returncode == 2
    assert cli("run", f, "--math", "double").returncode == 2
    assert cli("run").returncode == 2
    assert cli("frobnicate", f).returncode == 2
    assert cli("run", tmp_path / "missing.json").returncode == 2


def test_cuda_backend_fails_loudly_without_a_device(tmp_path):
    """No silent CPU fallback: without a GPU the CUDA backend errors out."""
    need_cli()
    import torch
    if torch.cuda.is_available():
        return
    f, rec = program_file(tmp_path, "adam_W4_N4096", "sched_program")
    p = cli("run", f, *dims_args(rec))
    assert p.returncode == 2 and "error" in p.stderr.lower()
