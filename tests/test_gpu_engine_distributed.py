"""GPU: the drop-in GpuEngine in DISTRIBUTED mode — one process per rank (here
W processes sharing one B200 through CUDA IPC: the code path of one process
per GPU over NVLink). Each process executes only its own rank of every plan
step (Engine::run's per-rank loop, runtime.hpp:287-296, becomes the process
grid); inputs come from the reference's gen_decl_values, the peer mappings
and the result assembly go through a world all-gather (gloo here). Every
process must return the reference Engine's digest and RunReport counters."""
import json
import os
import socket
from pathlib import Path

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
GOLD = Path(__file__).resolve().parent / "golden"

CASES = {
    2: ["adam_W2_N1024", "adam_W2_N4096", "mp_W2_B2_S8_H64", "pp_W2_N4096", "rooted_sum_W2_N1024"],
    4: ["adam_W4_N4096", "mp_W4_B2_S8_H64", "pp_W4_N4096", "rooted_max_W4_N1024"],
}


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _golden(name):
    for f in GOLD.glob("*_cases.json"):
        for rec in json.loads(f.read_text()):
            if rec.get("name") == name:
                return rec
    raise KeyError(name)


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    out = []
    try:
        import torch

        from paper_2105_05720_b200 import _lib
        from paper_2105_05720_b200.engine import BASE, SCHEDULED, GpuEngineSession, torch_allgather

        torch.cuda.set_device(0)
        ag = torch_allgather()
        for name in CASES[world]:
            rec = _golden(name)
            s = GpuEngineSession(rec["base_program"], sched_program=rec["sched_program"])
            s.gen(rec["seed"])
            for which, key, rkey in ((SCHEDULED, "engine_sched_digest", "report_sched"),
                                     (BASE, "engine_base_digest", "report_base")):
                s.run(rec["seed"], which, device=0, math=_lib.MATH_EXACT, rank=rank, world=world, allgather=ag)
                rep = s.report()
                ok = "%016x" % s.digest() == rec[key]
                for k in ("comm_bytes", "intergroup_bytes", "kernel_steps", "memory_elems"):
                    ok &= rep[k] == rec[rkey][k]
                out.append((name, which, ok, rep["lowering"]))
            s.close()
        # the per-tensor LAMB list programs (reference-evaluated arrays)
        lrec = next(r for r in json.loads((GOLD / "lamb_list_cases.json").read_text()) if r["W"] == world)
        arrs = np.load(GOLD / "lamb_list_results.npz")
        s = GpuEngineSession((GOLD / "lamb_list_program.json").read_text(),
                             sched_program=(GOLD / "lamb_list_fused_program.json").read_text(), dims={"W": world})
        s.gen(1)
        s.run(1, SCHEDULED, device=0, math=_lib.MATH_EXACT, rank=rank, world=world, allgather=ag)
        ok = True
        for i, n in enumerate(lrec["counts"]):
            for nm in ("p", "m", "v"):
                got, want = s.result(f"tensor:{nm}{i}", 0, n), arrs[f"W{world}_{nm}{i}"]
                d = np.abs(got.view(np.int32).astype(np.int64) - want.view(np.int32).astype(np.int64))
                ok &= int(d.max()) <= (1 if nm == "p" else 0)
        out.append(("lamb_list", SCHEDULED, ok, s.report()["lowering"]))
        s.close()
        q.put((rank, out, None))
    except Exception as e:  # report, don't hang the parent
        q.put((rank, out, repr(e)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_gpu_engine_distributed_reproduces_reference(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=600) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, out, err in res:
        assert err is None, (rank, err)
        assert len(out) == 2 * len(CASES[world]) + 1
        for name, which, ok, low in out:
            assert ok, f"rank {rank}: {name} ({'sched' if which == 0 else 'base'}) differs: {low}"
        low = " ".join(x for name, which, _, lw in out if which == 0 for x in lw)
        assert "fused_rs_adam_ag" in low and "rs_fused_send_ag" in low and "fused_rs_lamb_ag" in low
