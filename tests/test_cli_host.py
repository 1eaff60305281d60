"""coconet-ccopt on the host (no GPU): the reference CLI contract — the
subcommands that never touch the data path, the simulated backend reproducing
the reference Engine's golden digests, argument errors (exit 2), and that the
CUDA backend fails loudly without a device instead of falling back."""
import json
from pathlib import Path

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


def _write_tensor(base, name, arr):
    """The reference's tensor file (json_io.hpp:580-593): f32 .bin + JSON sidecar."""
    import numpy as np
    np.asarray(arr, dtype="<f4").tofile(str(base) + ".bin")
    (Path(str(base) + ".json")).write_text(json.dumps({"name": name, "shape": list(arr.shape), "elem": "f32"}))


def test_tensor_file_io_round_trip(tmp_path):
    """--input reads decls from tensor files, --dump writes every result array:
    feeding the values gen_decl_values would make reproduces the golden digest,
    and the dumped arrays hash to the report's per-key digests."""
    need_cli()
    import numpy as np

    from oracle import coconet_oracle as co
    f, rec = program_file(tmp_path, "adam_W4_N4096", "sched_program")
    W, N = rec["dims"]["W"], rec["dims"]["N"]
    p = co.gen_decl(1, "p", [N], "replicated", 0, W)
    m = co.gen_decl(1, "m", [N], "replicated", 0, W)  # global view of the sliced decl
    _write_tensor(tmp_path / "p", "p", np.asarray(p))
    _write_tensor(tmp_path / "m", "m", np.asarray(m))
    out = tmp_path / "dump"
    out.mkdir()
    j = json.loads(cli("run", f, *dims_args(rec), "--backend", "sim", "--input", f"p={tmp_path / 'p'}",
                       "--input", f"m={tmp_path / 'm'}", "--dump", out, check_rc=0).stdout)
    assert j["digest"] == rec["engine_sched_digest"]
    for key, summ in j["results"].items():
        stem = key.replace(":", "_").replace("/", "_")
        files = sorted(out.glob(f"{stem}_r*.bin"), key=lambda x: int(x.stem.rsplit("_r", 1)[1]))
        assert files, key
        h = co.FNV_OFFSET
        for fb in files:
            side = json.loads(fb.with_suffix(".json").read_text())
            assert side["name"] == key and side["elem"] == "f32"
            h = co.fnv1a(np.fromfile(fb, dtype="<f4").tobytes(), h)
        assert "%016x" % h == summ["digest"], key
    # a different p changes the result; a wrong shape is rejected
    _write_tensor(tmp_path / "p2", "p", np.asarray(p) * 2)
    j2 = json.loads(cli("run", f, *dims_args(rec), "--backend", "sim", "--input", f"p={tmp_path / 'p2'}",
                        check_rc=0).stdout)
    assert j2["digest"] != rec["engine_sched_digest"]
    _write_tensor(tmp_path / "bad", "p", np.zeros(7, np.float32))
    assert cli("run", f, *dims_args(rec), "--backend", "sim", "--input", f"p={tmp_path / 'bad'}").returncode == 2
