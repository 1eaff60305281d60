"""Small instances of every kernel family for compute-sanitizer (memcheck,
racecheck, synccheck): LAMB (GRID, TMA, STREAMED; W = 1..4; ONCHIP at W = 1,
also with a hold of 1 so windows, spills and the TMEM/shared-memory slot ring
all run), Adam (LDG, TMA at W = 1..3), tensor-list AllReduce,
Reduce/Broadcast, RS/AG, the MP epilogue, the tile-flag overlapped tcgen05
GEMM + all-reduce, the all-gather -> GEMM MP kernel (AUTO), the plain GEMM
(1-SM and the 2-SM pair kernel), and the PP send; the DP cases also on a
cuMem-backed heap.
Usage: compute-sanitizer --tool TOOL python tools/sanitize_cases.py"""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import (AdamHParams, BdrHParams, LambHParams, TensorList, all_gather,  # noqa: E402
                                               allreduce, broadcast, fused_rs_adam_ag, fused_rs_bdr_ag,
                                               fused_rs_lamb_ag, matmul, mm_overlap_fused_ar, reduce,
                                               reduce_scatter, rs_fused_send_ag)
from paper_2105_05720_b200.runtime import Context  # noqa: E402


def dp(W, cap, heap="default"):
    counts = [3000, 77, 5000, 1, 4096]
    ctx = Context(W, heap_bytes=32 << 20, timeout_ms=20000, heap=heap)
    tl = TensorList(ctx, counts, bucket_cap=cap)
    g = [ctx.alloc([n], torch.float16) for n in counts]
    p = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    for r in range(W):
        for i in range(len(counts)):
            ctx.view(g[i], r).normal_()
            ctx.view(p[i], r).uniform_(0.1, 0.9)
        ctx.view(m, r).zero_()
        ctx.view(v, r).fill_(1e-3)
    scheds = [_lib.LAMB_GRID, _lib.LAMB_STREAMED, _lib.LAMB_TMA] + ([_lib.LAMB_ONCHIP] if W == 1 else [])
    for sched in scheds:
        fused_rs_lamb_ag(ctx, tl, g, p, m, v, LambHParams(1e-3, 0.9, 0.999, 1.0, sched=sched, lag_elems=3000))
    if W == 1:  # ONCHIP with one held item per CTA: several windows, spilled items, slot-ring wrap
        os.environ["COCONET_LAMB_OC_HOLD"] = "1"
        os.environ["COCONET_LAMB_OC_STAGES"] = "2"
        try:
            tl2 = TensorList(ctx, counts, bucket_cap=cap)
            fused_rs_lamb_ag(ctx, tl2, g, p, m, v, LambHParams(1e-3, 0.9, 0.999, 1.0, sched=_lib.LAMB_ONCHIP))
        finally:
            os.environ.pop("COCONET_LAMB_OC_HOLD")
            os.environ.pop("COCONET_LAMB_OC_STAGES")
    for math in (_lib.MATH_EXACT, _lib.MATH_FAST):
        fused_rs_adam_ag(ctx, tl, g, p, m, v, AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, math, _lib.ALGO_TWO_SHOT))
    out = [ctx.alloc([n], torch.float16) for n in [3000, 77, 5000, 1, 4096]]
    allreduce(ctx, tl, g, out)
    ctx.check()
    ctx.close()


def rooted_axis(W):
    ctx = Context(W, heap_bytes=16 << 20, timeout_ms=20000)
    x, o = ctx.alloc([4096]), ctx.alloc([4096])
    for r in range(W):
        ctx.view(x, r).normal_()
    reduce(ctx, x, o, root=W - 1)
    broadcast(ctx, x, o, root=0)
    s = ctx.alloc([4096 // W])
    reduce_scatter(ctx, x, s, axis=0)
    all_gather(ctx, s, o, axis=0)
    ctx.check()
    ctx.close()


def mp_pp(W):
    rows, H = 256, 128 * W
    k = H // W
    dt = torch.bfloat16
    ctx = Context(W, heap_bytes=64 << 20, timeout_ms=20000)
    x, w = ctx.alloc([rows, k], dt), ctx.alloc([k, H], dt)
    part, bb, rr, out = ctx.alloc([rows, H], dt), ctx.alloc([H], dt), ctx.alloc([rows, H], dt), ctx.alloc([rows, H], dt)
    for r in range(W):
        ctx.view(x, r).normal_()
        ctx.view(w, r).normal_()
        ctx.view(bb, r).normal_()
        ctx.view(rr, r).normal_()
    hp = BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_FAST)
    matmul(ctx, x, w, part, math=_lib.MATH_FAST)
    fused_rs_bdr_ag(ctx, part, bb, rr, out, hp)
    os.environ["COCONET_MP_OVERLAP"] = "fused"
    mm_overlap_fused_ar(ctx, x, w, bb, rr, part, out, hp)
    os.environ.pop("COCONET_MP_OVERLAP")
    mm_overlap_fused_ar(ctx, x, w, bb, rr, part, out, hp)  # AUTO: all-gather -> GEMM at W >= 2
    if W >= 2:
        S = W // 2
        g0, g1 = ctx.group(0, S), ctx.group(S, S)
        N = 1024 * S
        xs, b2, r2, o2 = (ctx.alloc([N]) for _ in range(4))
        rs_fused_send_ag(ctx, g0, g1, xs, b2, r2, o2, BdrHParams(0.1, 1, 3251584743947114031, _lib.MATH_EXACT))
        xh, bh, rh, oh = (ctx.alloc([N], torch.float16) for _ in range(4))  # 16-byte vector path
        rs_fused_send_ag(ctx, g0, g1, xh, bh, rh, oh, BdrHParams(0.1, 1, 3251584743947114031, _lib.MATH_FAST))
    fused_rs_bdr_ag(ctx, part, bb, rr, out, BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_EXACT))
    ctx.check()
    ctx.close()


if __name__ == "__main__":
    for W, cap in ((1, 1024), (1, 4096), (2, 1024), (4, 512), (2, 16384), (3, 16384)):  # 16384: Adam TMA at W>1
        dp(W, cap)
    dp(2, 1024, heap="cumem")  # the cuMem-backed heap (csrc/heap_cumem.cu)
    for W in (2, 4):
        rooted_axis(W)
    for W in (1, 2, 4):
        mp_pp(W)
    print("sanitize cases done")
