"""GPU: the cuMem-backed symmetric heap (csrc/heap_cumem.cu) and the NVLS
gate. A cuMem heap must give bit-identical results to the cudaMalloc heap
(same offsets, same kernels); NVLS must report why it is unavailable and
fail loudly (Unsupported) when asked for without a multicast mapping - never
fall back to another algorithm silently. The multicast kernels themselves
need two or more NVSwitch-connected GPUs: test_nvls_* runs them when the box
has them and is skipped otherwise (one-GPU boxes, see
profiles/r02_nvls_probe.txt)."""
import numpy as np
import pytest
import torch

from oracle import coconet_oracle as co
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import (AdamHParams, LambHParams, TensorList, allreduce, fused_rs_adam_ag,
                                               fused_rs_lamb_ag)
from paper_2105_05720_b200.runtime import Context, nvls_supported
from tests.dp_util import DPWorkload, dsl_scalars

pytestmark = pytest.mark.gpu


def _adam_and_allreduce(heap, W, counts, math):
    ctx = Context(W, mode="virtual", heap_bytes=64 << 20, timeout_ms=5000, heap=heap)
    assert ctx.heap_kind == heap
    wl = DPWorkload(ctx, [sum(counts)])  # goldens/adam.json: one tensor
    wl.gen_dsl()
    sc = dsl_scalars(1, W)
    wl.adam(AdamHParams(lr=sc["lr"], beta1=sc["beta1"], beta2=sc["beta2"], t=sc["t"], math=math,
                        algo=_lib.ALGO_TWO_SHOT))
    ctx.check()
    p = [wl.params_host(r) for r in range(W)]
    m, v = wl.state_host()
    tl = TensorList(ctx, counts)
    xs = [ctx.alloc([n]) for n in counts]
    outs = [ctx.alloc([n]) for n in counts]
    rng = np.random.default_rng(5)
    xv = [[rng.uniform(-1, 1, n).astype(np.float32) for n in counts] for _ in range(W)]
    for r in range(W):
        for t, n in enumerate(counts):
            ctx.view(xs[t], r).copy_(torch.from_numpy(xv[r][t]))
    allreduce(ctx, tl, xs, outs)
    ctx.check()
    ar = [[ctx.view(o, r).cpu().numpy() for o in outs] for r in range(W)]
    ctx.close()
    return p, m, v, ar


@pytest.mark.parametrize("W", [2, 4])
@pytest.mark.parametrize("math", [_lib.MATH_EXACT, _lib.MATH_FAST])
def test_cumem_heap_bitwise_equals_cudamalloc_heap(W, math):
    counts = [3000, 1024, 77, 5000]
    a = _adam_and_allreduce("cudamalloc", W, counts, math)
    b = _adam_and_allreduce("cumem", W, counts, math)
    for x, y in zip(a[0], b[0]):  # gathered p on every rank
        assert all(np.array_equal(u, w) for u, w in zip(x, y))
    for x, y in zip(a[1] + a[2], b[1] + b[2]):  # m, v shards
        assert np.array_equal(x, y)
    for x, y in zip(a[3], b[3]):
        assert all(np.array_equal(u, w) for u, w in zip(x, y))


def test_cumem_heap_kind_from_environment(monkeypatch):
    monkeypatch.setenv("COCONET_HEAP", "cumem")
    ctx = Context(2, mode="virtual", heap_bytes=8 << 20)
    assert ctx.heap_kind == "cumem"
    # the heap is rounded to the allocation granularity, not below the request
    assert int(ctx.lib.coconet_heap_bytes(ctx.handle)) >= 8 << 20
    ctx.close()


def test_nvls_gate_reports_and_refuses():
    ok, why = nvls_supported(0, 2)
    if not ok:
        assert why  # the reason is stated (profiles/r02_nvls_probe.txt on one-GPU boxes)
    # an NVLS heap spans one GPU per process: refused in VIRTUAL mode
    with pytest.raises(_lib.CoconetError, match="Unsupported"):
        Context(2, mode="virtual", heap_bytes=8 << 20, heap="nvls")
    # ALGO_NVLS without a multicast mapping is an error, never a silent two-shot
    ctx = Context(2, mode="virtual", heap_bytes=16 << 20, timeout_ms=5000)
    assert not ctx.nvls
    wl = DPWorkload(ctx, [4096])
    wl.gen_dsl()
    sc = dsl_scalars(1, 2)
    with pytest.raises(_lib.CoconetError, match="Unsupported"):
        wl.adam(AdamHParams(lr=sc["lr"], beta1=sc["beta1"], beta2=sc["beta2"], t=sc["t"],
                            math=_lib.MATH_FAST, algo=_lib.ALGO_NVLS))
    with pytest.raises(_lib.CoconetError, match="Unsupported"):
        wl.lamb(LambHParams(lr=0.01, beta1=0.9, beta2=0.999, t=1.0, sched=_lib.LAMB_NVLS))
    tl = TensorList(ctx, [4096])
    x, o = [ctx.alloc([4096])], [ctx.alloc([4096])]
    with pytest.raises(_lib.CoconetError, match="Unsupported"):
        allreduce(ctx, tl, x, o, algo=_lib.ALGO_NVLS)
    ctx.close()


def _nvls_worker(rank, world, port, counts, q):
    import os

    import torch.distributed as dist

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(rank)
        ctx = Context(world, mode="distributed", rank=rank, device=rank, heap_bytes=64 << 20, timeout_ms=60000,
                      heap="nvls")
        assert ctx.nvls
        rng = np.random.default_rng(3)
        g = [rng.uniform(-1, 1, (world, n)).astype(np.float32) for n in counts]
        p = [rng.uniform(0.1, 0.9, n).astype(np.float32) for n in counts]
        tl = TensorList(ctx, counts)
        res = {}
        for algo in (_lib.ALGO_TWO_SHOT, _lib.ALGO_NVLS):
            gb = [ctx.alloc([n]) for n in counts]
            pb = [ctx.alloc([n]) for n in counts]
            mb, vb = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
            ob = [ctx.alloc([n]) for n in counts]
            for t in range(len(counts)):
                ctx.view(gb[t]).copy_(torch.from_numpy(g[t][rank]))
                ctx.view(pb[t]).copy_(torch.from_numpy(p[t]))
            ctx.view(mb).zero_()
            ctx.view(vb).zero_()
            torch.cuda.synchronize()
            dist.barrier()
            fused_rs_adam_ag(ctx, tl, gb, pb, mb, vb, AdamHParams(0.01, 0.9, 0.999, 1.0, 0.0, True,
                                                                   _lib.MATH_FAST, algo))
            allreduce(ctx, tl, gb, ob, algo=algo)
            ctx.check()
            got_p = [ctx.view(b).cpu().numpy() for b in pb]
            # LAMB: GRID across ranks against its NVLS schedule
            for t in range(len(counts)):
                ctx.view(pb[t]).copy_(torch.from_numpy(p[t]))
            ctx.view(mb).zero_()
            ctx.view(vb).zero_()
            torch.cuda.synchronize()
            dist.barrier()
            fused_rs_lamb_ag(ctx, tl, gb, pb, mb, vb, LambHParams(
                lr=0.01, beta1=0.9, beta2=0.999, t=1.0,
                sched=_lib.LAMB_NVLS if algo == _lib.ALGO_NVLS else _lib.LAMB_GRID))
            ctx.check()
            res[algo] = (got_p, [ctx.view(b).cpu().numpy() for b in ob], [ctx.view(b).cpu().numpy() for b in pb])
        dev = max(co.max_rel_deviation(a, b) for k in (0, 1, 2)
                  for a, b in zip(res[_lib.ALGO_NVLS][k], res[_lib.ALGO_TWO_SHOT][k]))
        dist.barrier()
        ctx.close()
        q.put((rank, dev, None))
    except Exception as e:  # report, don't hang the parent
        q.put((rank, 1.0, repr(e)))
    finally:
        dist.destroy_process_group()


def test_nvls_adam_and_allreduce_match_two_shot():
    """COCONET_ALGO_NVLS / COCONET_LAMB_NVLS (multimem.ld_reduce RS +
    multimem.st AG) within fp32 rounding of the P2P two-shot, one process per
    GPU: fused Adam, AllReduce and fused LAMB."""
    import socket

    import torch.multiprocessing as mp

    world = torch.cuda.device_count()
    ok, why = nvls_supported(0, max(world, 2))
    if world < 2 or not ok:
        pytest.skip(f"NVLS needs >= 2 NVSwitch-connected GPUs with multicast: {why or 'one GPU'}")
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    counts = [3000, 1024, 77, 5000]
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_nvls_worker, args=(r, world, port, counts, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
    for rank, dev, err in res:
        assert err is None, err
        assert dev <= 1e-5, f"rank {rank}: NVLS deviates {dev} from two-shot"
