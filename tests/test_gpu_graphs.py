"""GPU: the fused calls captured in a CUDA graph and replayed (the small-
message path: C1's 2^20-element Adam is launch-bound from Python, DESIGN.md
§5.2c). A replay must equal the same number of eager calls bit for bit —
including kernels with a mid-kernel cross-rank barrier (LAMB's norm
exchange), whose flag protocol resets consumed slots so the epoch baked
into the captured launch stays valid (common.cuh rank_barrier) — in VIRTUAL
mode and across processes (DISTRIBUTED, two processes sharing one B200)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import AdamHParams, LambHParams, TensorList, allreduce
from tests.dp_util import DPWorkload, new_ctx

pytestmark = pytest.mark.gpu

COUNTS = [3000, 1024, 77, 5000, 20_000]


def _inputs(W, seed=5):
    rng = np.random.default_rng(seed)
    g = [rng.uniform(-1, 1, (W, n)).astype(np.float32) for n in COUNTS]
    p = [rng.uniform(0.1, 0.9, n).astype(np.float32) for n in COUNTS]
    m = [rng.uniform(-0.1, 0.1, n).astype(np.float32) for n in COUNTS]
    v = [rng.uniform(0.01, 0.2, n).astype(np.float32) for n in COUNTS]
    return g, p, m, v


def _run(W, step_fn, graph, replays=3, cap=1024):
    ctx = new_ctx(W)
    wl = DPWorkload(ctx, COUNTS, bucket_cap=cap)
    wl.set_host(*_inputs(W))
    step_fn(wl)  # eager warm-up: bucket tables, occupancy and smem attributes cached
    ctx.check()
    if graph:
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            with torch.cuda.graph(g, stream=s):
                step_fn(wl)
        torch.cuda.current_stream().wait_stream(s)
        for _ in range(replays):
            g.replay()
    else:
        for _ in range(replays):
            step_fn(wl)
    ctx.check()
    out = [wl.params_host(r) for r in range(W)], wl.state_host()
    ctx.close()
    return out


def _same(a, b):
    (pa, (ma, va)), (pb, (mb, vb)) = a, b
    for t in range(len(COUNTS)):
        assert np.array_equal(ma[t], mb[t]) and np.array_equal(va[t], vb[t])
        for r in range(len(pa)):
            assert np.array_equal(pa[r][t], pb[r][t])


@pytest.mark.parametrize("W", [1, 4])
@pytest.mark.parametrize("math", [_lib.MATH_EXACT, _lib.MATH_FAST])
def test_adam_graph_replay_equals_eager(W, math):
    hp = AdamHParams(0.01, 0.9, 0.999, 2.0, 1e-8, False, math, _lib.ALGO_TWO_SHOT)
    f = lambda wl: wl.adam(hp)  # noqa: E731
    _same(_run(W, f, True), _run(W, f, False))


@pytest.mark.parametrize("W,cap,sched", [(1, 16384, _lib.LAMB_TMA), (1, 16384, _lib.LAMB_ONCHIP),
                                         (4, 1024, _lib.LAMB_GRID),
                                         (4, 16384, _lib.LAMB_TMA)])
def test_lamb_graph_replay_equals_eager(W, cap, sched):
    """LAMB has a real cross-rank barrier mid-kernel (the norm exchange)."""
    hp = LambHParams(lr=0.01, beta1=0.9, beta2=0.999, t=2.0, sched=sched)
    f = lambda wl: wl.lamb(hp)  # noqa: E731
    _same(_run(W, f, True, cap=cap), _run(W, f, False, cap=cap))


def test_allreduce_graph_replay():
    W = 4
    ctx = new_ctx(W)
    tl = TensorList(ctx, COUNTS)
    xs = [ctx.alloc([n]) for n in COUNTS]
    outs = [ctx.alloc([n]) for n in COUNTS]
    for t, n in enumerate(COUNTS):
        for r in range(W):
            ctx.view(xs[t], r).fill_(float(r + 1))
    allreduce(ctx, tl, xs, outs)
    ctx.check()
    for t in range(len(COUNTS)):
        for r in range(W):
            ctx.view(outs[t], r).zero_()
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            allreduce(ctx, tl, xs, outs)
    torch.cuda.current_stream().wait_stream(s)
    g.replay()
    g.replay()
    ctx.check()
    for t in range(len(COUNTS)):
        for r in range(W):
            assert torch.all(ctx.view(outs[t], r) == 10.0)  # 1 + 2 + 3 + 4 (test_runtime.cpp:28-37)
    ctx.close()


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_2105_05720_b200.collectives import fused_rs_adam_ag, fused_rs_lamb_ag
        from paper_2105_05720_b200.runtime import Context

        torch.cuda.set_device(0)
        res = {}
        for kind in ("adam", "lamb"):
            outs = []
            for graph in (True, False):
                ctx = Context(world, mode="distributed", rank=rank, device=0, heap_bytes=64 << 20, timeout_ms=60000)
                tl = TensorList(ctx, COUNTS)
                g, p, m, v = _inputs(world, 7)
                gb = [ctx.alloc([n]) for n in COUNTS]
                pb = [ctx.alloc([n]) for n in COUNTS]
                mb, vb = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
                for t in range(len(COUNTS)):
                    ctx.view(gb[t]).copy_(torch.from_numpy(g[t][rank]))
                    ctx.view(pb[t]).copy_(torch.from_numpy(p[t]))
                ctx.view(mb).zero_()
                ctx.view(vb).fill_(0.01)
                torch.cuda.synchronize()
                dist.barrier()
                if kind == "adam":
                    hp = AdamHParams(0.01, 0.9, 0.999, 2.0, 1e-8, False, _lib.MATH_EXACT, _lib.ALGO_TWO_SHOT)
                    step = lambda: fused_rs_adam_ag(ctx, tl, gb, pb, mb, vb, hp)  # noqa: E731
                else:
                    hp = LambHParams(lr=0.01, beta1=0.9, beta2=0.999, t=2.0, sched=_lib.LAMB_GRID)
                    step = lambda: fused_rs_lamb_ag(ctx, tl, gb, pb, mb, vb, hp)  # noqa: E731
                step()
                ctx.check()
                if graph:
                    cg = torch.cuda.CUDAGraph()
                    s = torch.cuda.Stream()
                    s.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(s):
                        with torch.cuda.graph(cg, stream=s):
                            step()
                    torch.cuda.current_stream().wait_stream(s)
                    torch.cuda.synchronize()
                    dist.barrier()
                    for _ in range(3):
                        cg.replay()
                else:
                    for _ in range(3):
                        step()
                ctx.check()
                outs.append(torch.cat([ctx.view(b) for b in pb] + [ctx.view(mb), ctx.view(vb)]).cpu())
                torch.cuda.synchronize()
                dist.barrier()
                ctx.close()
            res[kind] = bool(torch.equal(outs[0], outs[1]))
        q.put((rank, res, None))
    except Exception as e:
        q.put((rank, {}, repr(e)))
    finally:
        dist.destroy_process_group()


def test_distributed_graph_replay_equals_eager():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, r, err in res:
        assert err is None, (rank, err)
        assert r == {"adam": True, "lamb": True}, (rank, r)
