"""Kernel-level timing probe (not the bench): per-kernel CUDA-event times of
the fused DP kernels at BERT-336M size on one GPU, next to a torch copy as the
bandwidth yardstick. Usage: python tools/probe.py [--steps K]"""
import argparse
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import (AdamHParams, LambHParams, TensorList, allreduce,  # noqa: E402
                                               fused_rs_adam_ag, fused_rs_lamb_ag, gen_values)
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from paper_2105_05720_b200.workloads import bert_large_counts  # noqa: E402


def timeit(fn, steps):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--only", default="")
    ap.add_argument("--cap", type=int, default=1024)
    args = ap.parse_args()
    counts = bert_large_counts()
    N = sum(counts)
    out = {}
    a = torch.empty(N, dtype=torch.float32, device="cuda")
    b = torch.empty_like(a)
    ms = timeit(lambda: b.copy_(a), args.steps)
    out["torch_copy_f32"] = {"ms": ms, "GBs": 8 * N / ms / 1e6}
    del a, b
    for W in (1,):
        ctx = Context(W, heap_bytes=sum(counts) * 24 + (1 << 30))
        tl = TensorList(ctx, counts, bucket_cap=args.cap)
        for gdt, gname in ((torch.float16, "f16"), (torch.float32, "f32")):
            grads = [ctx.alloc([n], gdt) for n in counts]
            params = [ctx.alloc([n]) for n in counts]
            m = ctx.alloc([tl.shard_elems])
            v = ctx.alloc([tl.shard_elems])
            for r in range(W):
                for i, n in enumerate(counts):
                    gen_values(ctx, ctx.view(grads[i], r), 1, f"g{i}", "local", r, [n], group_size=W)
                    gen_values(ctx, ctx.view(params[i], r), 1, f"p{i}", "replicated", r, [n], group_size=W)
                ctx.view(m, r).fill_(0.0)
                ctx.view(v, r).fill_(1e-3)
            gb = 2 if gdt == torch.float16 else 4
            hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0)
            byt = (gb + 12 + 8 + 12 + 4) * N
            for sched, sn in ((_lib.LAMB_GRID, "grid"), (_lib.LAMB_TMA, "tma")):
                hps = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched)
                ms = timeit(lambda: fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hps), args.steps)
                out[f"lamb_W{W}_g{gname}_{sn}"] = {"ms": ms, "GBs": byt / ms / 1e6, "bytes": byt}
            for math, mn in ((_lib.MATH_FAST, "fast"), (_lib.MATH_EXACT, "exact")):
                hpa = AdamHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, eps=1e-8, math=math,
                                  algo=_lib.ALGO_TWO_SHOT)
                ms = timeit(lambda: fused_rs_adam_ag(ctx, tl, grads, params, m, v, hpa), args.steps)
                byt = (gb + 12 + 12) * N
                out[f"adam_W{W}_g{gname}_{mn}"] = {"ms": ms, "GBs": byt / ms / 1e6, "bytes": byt}
            outs = [ctx.alloc([n], gdt) for n in counts]
            ms = timeit(lambda: allreduce(ctx, tl, grads, outs), args.steps)
            out[f"allreduce_W{W}_{gname}"] = {"ms": ms, "GBs": 2 * gb * N / ms / 1e6}
            ctx.reset()
        ctx.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__" and not os.environ.get("PROBE_EXTRA"):
    main()


def extra_probes(steps=10):
    """LAMB bucket-capacity sensitivity; torch's fused multi-tensor Adam on the
    same list (library baseline); C5 = 3.9e9-parameter Adam at W=1."""
    out = {}
    counts = bert_large_counts()
    N = sum(counts)
    ctx = Context(1, heap_bytes=N * 24 + (1 << 30))
    for cap in (1024, 4096, 16384, 32768, 65536):
        tl = TensorList(ctx, counts, bucket_cap=cap)
        grads = [ctx.alloc([n], torch.float16) for n in counts]
        params = [ctx.alloc([n]) for n in counts]
        m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
        for i, n in enumerate(counts):
            ctx.view(grads[i], 0).normal_()
            ctx.view(params[i], 0).uniform_(0.1, 0.9)
        ctx.view(m, 0).zero_()
        ctx.view(v, 0).fill_(1e-3)
        hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0)
        ms = timeit(lambda: fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp), steps)
        out[f"lamb_cap{cap}_ms"] = ms
        tl.close()
        ctx.reset()
    ctx.close()
    # torch fused multi-tensor Adam (fp32 grads/params/state), same 398 tensors
    ps = [torch.rand(n, device="cuda") for n in counts]
    gs = [torch.randn(n, device="cuda") for n in counts]
    ms_ = [torch.zeros(n, device="cuda") for n in counts]
    vs_ = [torch.full((n,), 1e-3, device="cuda") for n in counts]
    steps_t = [torch.tensor(1.0, device="cuda") for _ in counts]
    f = lambda: torch._fused_adam_(ps, gs, ms_, vs_, [], steps_t, amsgrad=False, lr=1e-3, beta1=0.9,
                                   beta2=0.999, weight_decay=0.0, eps=1e-8, maximize=False)
    out["torch_fused_adam_fp32_ms"] = timeit(f, steps)
    del ps, gs, ms_, vs_
    torch.cuda.empty_cache()
    # C5 at W=1: 3.9e9 parameters, fp32 grads/params/state (64-bit indexing)
    n5 = 3_900_000_000
    ctx = Context(1, heap_bytes=n5 * 16 + (1 << 30))
    tl = TensorList(ctx, [n5])
    g, p = ctx.alloc([n5]), ctx.alloc([n5])
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    gen_values(ctx, ctx.view(g, 0), 1, "g", "local", 0, [n5], group_size=1)
    gen_values(ctx, ctx.view(p, 0), 1, "p", "replicated", 0, [n5], group_size=1)
    ctx.view(m, 0).zero_()
    ctx.view(v, 0).fill_(1e-3)
    hp = AdamHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, eps=1e-8, math=_lib.MATH_FAST, algo=_lib.ALGO_TWO_SHOT)
    ms = timeit(lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp), 5)
    out["c5_adam_3.9e9_W1_fast_ms"] = ms
    out["c5_adam_GBs"] = 28 * n5 / (ms * 1e-3) / 1e9
    ctx.close()
    return out


if __name__ == "__main__" and os.environ.get("PROBE_EXTRA"):
    print(json.dumps(extra_probes(), indent=1))
