"""Per-pattern timing on ONE GPU with virtual ranks (all W ranks' data in this
device's HBM; "NVLink" traffic becomes local HBM traffic, so these are kernel
and protocol costs, not link-bound numbers). Configs from BASELINE.json:
  C1  Adam 2^20 fp32, W=4          (fused RS-Adam-AG, exact and fast)
  C3  MP [8192x384]x[384x3072] bf16, W=8 (tcgen05 GEMM, fused RS-BDR-AG, overlap)
  C4  PP N=25,165,824, 2 stages x 4 (RS -> fused send -> AG)
Usage: python tools/pattern_probe.py [--only c1,c3,c4] [--gemm-only]"""
import argparse
import os
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import (AdamHParams, BdrHParams, TensorList, fused_rs_adam_ag,  # noqa: E402
                                               fused_rs_bdr_ag, gen_values, matmul, mm_overlap_fused_ar,
                                               rs_fused_send_ag)
from paper_2105_05720_b200.runtime import Context  # noqa: E402


def timeit(fn, steps=20, warmup=3):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / steps


def devtime(fn, steps=20, warmup=3, flush_bytes=0):
    """Device time of one call, without the host's launch gaps: each call is
    queued behind a ~25 us device sleep, so the kernel starts the moment its
    start event completes. flush_bytes > 0 writes that many bytes between
    calls (outside the events) so every call starts with a cold L2."""
    for _ in range(warmup):
        fn()
    scratch = torch.empty(flush_bytes // 4, dtype=torch.float32, device="cuda") if flush_bytes else None
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
    torch.cuda.synchronize()
    for e0, e1 in ev:
        if scratch is not None:
            scratch.zero_()
        torch.cuda._sleep(50_000)
        e0.record()
        fn()
        e1.record()
    torch.cuda.synchronize()
    return sum(e0.elapsed_time(e1) for e0, e1 in ev) / steps


def c1(out):
    W, N = 4, 1 << 20
    ctx = Context(W, heap_bytes=64 << 20)
    tl = TensorList(ctx, [N])
    g, p = ctx.alloc([N]), ctx.alloc([N])
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    for r in range(W):
        gen_values(ctx, ctx.view(g, r), 1, "g", "local", r, [N], group_size=W)
        gen_values(ctx, ctx.view(p, r), 1, "p", "replicated", r, [N], group_size=W)
        ctx.view(m, r).zero_()
        ctx.view(v, r).fill_(1e-3)
    for math, name in ((_lib.MATH_EXACT, "exact"), (_lib.MATH_FAST, "fast")):
        for algo, an in ((_lib.ALGO_TWO_SHOT, "two_shot"),):
            hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 0.0, True, math, algo)
            f = lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp)  # noqa: E731
            # per call from Python, back to back (host-bound at this size)
            out[f"c1_adam_W4_N2^20_{name}_{an}_us"] = timeit(f, 50) * 1e3
            # the kernel alone, L2 flushed before each call (512 MB write)
            dev = devtime(f, 20, flush_bytes=512 << 20)
            out[f"c1_adam_W4_N2^20_{name}_{an}_device_cold_us"] = dev * 1e3
            # HBM bytes of all W ranks here: each pulls its chunk of g from W
            # ranks and pushes p to W ranks (8N), plus m, v, p read and m, v
            # written on its own chunk (20N/W): (8W + 20) N in total
            out[f"c1_adam_W4_N2^20_{name}_{an}_device_cold_GBs"] = (8 * W + 20) * N / (dev * 1e-3) / 1e9
            # the same call captured in a CUDA graph, 20 calls per replay:
            # no Python or C-ABI host time per call (the small-message floor)
            gr = torch.cuda.CUDAGraph()
            st = torch.cuda.Stream()
            st.wait_stream(torch.cuda.current_stream())
            with torch.cuda.stream(st):
                with torch.cuda.graph(gr, stream=st):
                    for _ in range(20):
                        f()
            torch.cuda.current_stream().wait_stream(st)
            out[f"c1_adam_W4_N2^20_{name}_{an}_graph_us"] = timeit(gr.replay, 10) * 1e3 / 20
    ctx.close()


def c3(out, gemm_only=False):
    W, rows, H = 8, 8192, 3072
    k = H // W
    dt = torch.bfloat16
    ctx = Context(W, heap_bytes=(3 << 30))
    x, w = ctx.alloc([rows, k], dt), ctx.alloc([k, H], dt)
    part, bb, rr, o1 = ctx.alloc([rows, H], dt), ctx.alloc([H], dt), ctx.alloc([rows, H], dt), ctx.alloc([rows, H], dt)
    for r in range(W):
        ctx.view(x, r).normal_()
        ctx.view(w, r).normal_(0, k ** -0.5)
        ctx.view(bb, r).normal_(0, 0.1)
        ctx.view(rr, r).normal_()
    hp = BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_FAST)
    gemm = timeit(lambda: matmul(ctx, x, w, part, math=_lib.MATH_FAST))
    flops = 2.0 * rows * H * k * W
    out["c3_gemm_8ranks_us"] = gemm * 1e3
    out["c3_gemm_tflops"] = flops / (gemm * 1e-3) / 1e12
    if gemm_only:
        return
    ar = timeit(lambda: fused_rs_bdr_ag(ctx, part, bb, rr, o1, hp))
    out["c3_fused_rs_bdr_ag_exact_8ranks_us"] = timeit(
        lambda: fused_rs_bdr_ag(ctx, part, bb, rr, o1, BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_EXACT))) * 1e3
    ov = timeit(lambda: mm_overlap_fused_ar(ctx, x, w, bb, rr, part, o1, hp))
    os.environ["COCONET_MP_OVERLAP"] = "fused"  # the one-kernel overlap, forced
    ovf = timeit(lambda: mm_overlap_fused_ar(ctx, x, w, bb, rr, part, o1, hp))
    os.environ.pop("COCONET_MP_OVERLAP")
    out["c3_fused_rs_bdr_ag_8ranks_us"] = ar * 1e3
    out["c3_sequential_us"] = (gemm + ar) * 1e3
    out["c3_overlap_auto_us"] = ov * 1e3  # AUTO: the all-gather -> GEMM kernel
    out["c3_overlap_auto_tflops"] = flops / (ov * 1e-3) / 1e12
    out["c3_overlap_speedup_vs_sequential"] = (gemm + ar) / ov
    out["c3_overlap_fused_kernel_us"] = ovf * 1e3  # the tile-flag one-kernel overlap, forced
    # bytes the RS->epilogue->AG moves through HBM here (all 8 ranks): each rank
    # reads its column block from 8 partials, b and r, and writes the block to 8 outs
    blk = rows * (H // W) * 2
    out["c3_fused_ar_GBs"] = W * (8 * blk + blk + 8 * blk) / (ar * 1e-3) / 1e9
    ctx.close()


def c4(out):
    W, N = 8, 25_165_824
    S = W // 2
    ctx = Context(W, heap_bytes=(1 << 30))
    g0, g1 = ctx.group(0, S), ctx.group(S, S)
    x, bb, rr, o = (ctx.alloc([N]) for _ in range(4))
    for r in range(S):
        gen_values(ctx, ctx.view(x, r), 1, "in", "local", r, [N], group_size=S)
        gen_values(ctx, ctx.view(bb, r), 1, "b", "replicated", r, [N], group_size=S)
        gen_values(ctx, ctx.view(rr, r), 1, "r", "replicated", r, [N], group_size=S)
    for math, name in ((_lib.MATH_EXACT, "exact"), (_lib.MATH_FAST, "fast")):
        hp = BdrHParams(0.1, 1, 3251584743947114031, math)
        ms = timeit(lambda: rs_fused_send_ag(ctx, g0, g1, x, bb, rr, o, hp))
        out[f"c4_pp_2x4_N25M_fp32_{name}_us"] = ms * 1e3
        # HBM bytes on this device: each sender reads its chunk from 4 ranks + b + r,
        # writes it to 4 receivers: (4 + 2 + 4) * N/4 * 4B per sender, 4 senders
        out[f"c4_pp_{name}_GBs"] = 10 * N * 4 / (ms * 1e-3) / 1e9
    # fp16 activations (the paper's C4 runs fp16 as well)
    xh, bh, rh, oh = (ctx.alloc([N], torch.float16) for _ in range(4))
    for r in range(S):
        ctx.view(xh, r).copy_(ctx.view(x, r))
        ctx.view(bh, r).copy_(ctx.view(bb, r))
        ctx.view(rh, r).copy_(ctx.view(rr, r))
    hp = BdrHParams(0.1, 1, 3251584743947114031, _lib.MATH_FAST)
    ms = timeit(lambda: rs_fused_send_ag(ctx, g0, g1, xh, bh, rh, oh, hp))
    out["c4_pp_2x4_N25M_fp16_fast_us"] = ms * 1e3
    out["c4_pp_fp16_fast_GBs"] = 10 * N * 2 / (ms * 1e-3) / 1e9
    ctx.close()


def c5(out, n=3_900_000_000):
    """C5's optimizer step on ONE GPU: the whole 3.9e9-parameter fused Adam
    (fp32 g, p, m, v: 62 GB resident, 16384-element buckets -> the TMA ring).
    At W=8 each GPU applies 1/8 of it and pulls/pushes the rest over NVLink."""
    ctx = Context(1, heap_bytes=n * 16 + (1 << 30))
    tl = TensorList(ctx, [n], bucket_cap=16384)
    g, p = ctx.alloc([n]), ctx.alloc([n])
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    gen_values(ctx, ctx.view(g, 0), 1, "g", "local", 0, [n], group_size=1)
    gen_values(ctx, ctx.view(p, 0), 1, "p", "replicated", 0, [n], group_size=1)
    ctx.view(m, 0).zero_()
    ctx.view(v, 0).fill_(1e-3)
    hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, _lib.MATH_FAST, _lib.ALGO_TWO_SHOT)
    ms = timeit(lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp), 5)
    out["c5_adam_3.9e9_W1_fp32_ms"] = ms
    out["c5_adam_3.9e9_W1_GBs"] = 28 * n / ms / 1e6  # g 4 + m, v, p 12 read + m, v, p 12 written
    ctx.close()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--only", default="c1,c3,c4,c5")
    ap.add_argument("--gemm-only", action="store_true")
    a = ap.parse_args()
    out = {}
    sel = a.only.split(",")
    if "c1" in sel:
        c1(out)
    if "c5" in sel:
        c5(out)
    if "c3" in sel:
        c3(out, a.gemm_only)
    if "c4" in sel:
        c4(out)
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()


def unfused_baselines(out, steps=5):
    """The unfused GPU baseline at N=1 (north star: "NCCL plus separate
    kernels"; one GPU has no collective): the same LAMB step written with
    torch's multi-tensor _foreach kernels over the same 398 BERT-336M tensors
    (fp16 grads widened, fp32 p/m/v), and torch._fused_adam_ for Adam."""
    from paper_2105_05720_b200.workloads import bert_large_counts
    counts = bert_large_counts()
    dev = "cuda"
    g16 = [torch.randn(n, device=dev, dtype=torch.float16) for n in counts]
    p = [torch.rand(n, device=dev) for n in counts]
    m = [torch.zeros(n, device=dev) for n in counts]
    v = [torch.full((n,), 1e-3, device=dev) for n in counts]
    lr, b1, b2, eps, wd, t = 1e-3, 0.9, 0.999, 1e-6, 0.01, 1.0
    bc1, bc2 = 1 - b1 ** t, 1 - b2 ** t

    def lamb_step():
        g = [x.float() for x in g16]
        torch._foreach_mul_(m, b1)
        torch._foreach_add_(m, g, alpha=1 - b1)
        torch._foreach_mul_(v, b2)
        torch._foreach_addcmul_(v, g, g, value=1 - b2)
        den = torch._foreach_div(v, bc2)
        torch._foreach_sqrt_(den)
        torch._foreach_add_(den, eps)
        u = torch._foreach_div(m, bc1)
        torch._foreach_div_(u, den)
        torch._foreach_add_(u, p, alpha=wd)
        pn = torch._foreach_norm(p)
        un = torch._foreach_norm(u)
        ratio = [lr * a / b for a, b in zip(pn, un)]
        torch._foreach_mul_(u, ratio)
        torch._foreach_sub_(p, u)

    ms = timeit(lamb_step, steps)
    out["unfused_torch_foreach_lamb_bert336m_ms"] = ms
    del g16
    g32 = [torch.randn(n, device=dev) for n in counts]
    steps_t = [torch.tensor(1.0, device=dev) for _ in counts]
    f = lambda: torch._fused_adam_(p, g32, m, v, [], steps_t, amsgrad=False, lr=1e-3, beta1=0.9, beta2=0.999,
                                   weight_decay=0.0, eps=1e-8, maximize=False)
    out["unfused_torch_fused_adam_bert336m_fp32_ms"] = timeit(f, steps)


def c2_w8(out, steps=5):
    """The headline step at W=8 with VIRTUAL ranks: the LAMB kernel the
    8-GPU run uses (AUTO = the TMA ring for the local m/v/p, RS pulls of fp16
    g from 8 ranks, sharded m/v, AG pushes of p into 8 ranks), with all
    traffic in this GPU's HBM. Bytes per global
    element summed over ranks: every rank's g read once (8 x 2 B), pass 1
    m, v, p read + m, v written (20 B), pass 2 m, v, p read (12 B), p pushed
    into 8 copies (32 B) = 80 B."""
    from paper_2105_05720_b200.collectives import LambHParams, fused_rs_lamb_ag
    from paper_2105_05720_b200.workloads import bert_large_counts
    W = 8
    counts = bert_large_counts()
    N = sum(counts)
    ctx = Context(W, heap_bytes=N * 6 + 2 * (N // W + 64 * len(counts) + 4096) * 4 + (512 << 20))
    tl = TensorList(ctx, counts, bucket_cap=16384)
    grads = [ctx.alloc([n], torch.float16) for n in counts]
    params = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    for r in range(W):
        for i, n in enumerate(counts):
            ctx.view(grads[i], r).normal_()
            ctx.view(params[i], r).uniform_(0.1, 0.9)
        ctx.view(m, r).zero_()
        ctx.view(v, r).fill_(1e-3)
    hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0)
    ms = timeit(lambda: fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp), steps, warmup=2)
    out["c2_lamb_W8_virtual_ms"] = ms
    out["c2_lamb_W8_virtual_GBs"] = 80 * N / ms / 1e6
    ctx.close()
