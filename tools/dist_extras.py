"""The other BASELINE.json configs measured by `bench.py --gpus N` (N > 1), one
process per GPU in DISTRIBUTED mode (peers mapped over NVLink), each next to
its NCCL + separate-kernel baseline on the same GPUs (north star: "beats the
NCCL-plus-separate-kernels baseline on the same box"):

  C1  Adam 2^20 fp32 over the N ranks: fused RS-Adam-AG (two-shot and
      one-shot) vs all_reduce + torch._fused_adam_ and vs reduce_scatter +
      torch._fused_adam_ on the shard + all_gather
  C3  MP layer [8192 x 3072/N] x [3072/N x 3072] bf16: tcgen05 GEMM + fused
      RS-bias-dropout-residual-AG (one-kernel overlap and back-to-back) vs
      cuBLAS matmul + all_reduce + a torch epilogue
  C4  PP boundary, 2 stages of N/2, N = 25,165,824 fp16 and fp32:
      rs_fused_send_ag vs stage all_reduce + torch epilogue + send/recv of the
      slice + stage all_gather
  C5  Adam over 3.9e9 parameters (fp32, data parallel): fused RS-Adam-AG vs
      all_reduce + torch._fused_adam_ (replicated state)

Every time is CUDA events on each rank, max over ranks. Each entry carries
its NVLink bytes per rank per direction (= the reference's
comm_bytes) and the fraction of the per-direction peak. Collective: every
rank calls every function in the same order; rank 0 reports.

COCONET_SHARE_DEVICE=1 (a test mode: every rank on GPU 0, gloo instead of
NCCL) runs the same code with C5 scaled down, so the path is exercised on a
one-GPU box; its numbers mean nothing.
"""
from __future__ import annotations

import os
import sys
import traceback
from pathlib import Path

import torch
import torch.distributed as dist

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import (AdamHParams, BdrHParams, TensorList, fused_rs_adam_ag,  # noqa: E402
                                               mm_overlap_fused_ar, rs_fused_send_ag)

C5_PARAMS = 3_900_000_000
C4_N = 25_165_824


def share_mode() -> bool:
    return os.environ.get("COCONET_SHARE_DEVICE") == "1"


def max_over(x: float) -> float:
    t = torch.tensor([float(x)], dtype=torch.float64)
    if dist.get_backend() == "nccl":
        t = t.cuda()
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def dtime(fn, steps=10, warmup=3):
    """ms per call: CUDA events on this rank's stream, barrier on both sides,
    max over ranks."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(steps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    dist.barrier()
    return max_over(e0.elapsed_time(e1) / steps)


def _try(out, key, fn):
    try:
        out[key] = fn()
    except Exception as e:  # a baseline that cannot run here is reported, never fatal
        traceback.print_exc(file=sys.stderr)
        out[key] = {"failed": repr(e)[:300]}


def peer_copy_gbs(ctx, nbytes=1 << 30):
    """Each rank pulls nbytes from the next rank's heap into its own (one
    NVLink direction per GPU); GB/s per rank, min over ranks."""
    W, r = ctx.world, ctx.rank
    buf = ctx.alloc([nbytes // 4], torch.float32)
    dst = ctx.alloc([nbytes // 4], torch.float32)
    ctx.view(buf).fill_(1.0)
    torch.cuda.synchronize()
    dist.barrier()
    src = ctx.view(buf, (r + 1) % W)
    ms = dtime(lambda: ctx.view(dst).copy_(src), steps=10)
    ctx.free(dst)
    ctx.free(buf)
    return nbytes / (ms * 1e-3) / 1e9


def c1(ctx, out, nvl_peak):
    W, N = ctx.world, 1 << 20
    tl = TensorList(ctx, [N])
    g, p = ctx.alloc([N]), ctx.alloc([N])
    m, v = ctx.alloc([tl.state_elems]), ctx.alloc([tl.state_elems])
    ctx.view(g).normal_()
    ctx.view(p).uniform_(0.1, 0.9)
    ctx.view(m).zero_()
    ctx.view(v).fill_(1e-3)
    nvl = 2 * (W - 1) / W * N * 4
    res = {"workload": f"Adam 2^20 fp32, W={W}", "nvlink_bytes_per_rank_dir": nvl}
    for math, mn in ((_lib.MATH_FAST, "fast"), (_lib.MATH_EXACT, "exact")):
        for algo, an in ((_lib.ALGO_TWO_SHOT, "two_shot"), (_lib.ALGO_ONE_SHOT, "one_shot")):
            hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, math, algo)
            ms = dtime(lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp), steps=50)
            res[f"fused_{mn}_{an}_us"] = ms * 1e3
            if an == "two_shot":
                res[f"fused_{mn}_{an}_nvlink_frac"] = nvl / (ms * 1e-3) / 1e9 / nvl_peak
    ctx.check()
    # NCCL + separate kernel
    gt = ctx.view(g).clone()
    pt, mt, vt = ctx.view(p).clone(), torch.zeros(N, device="cuda"), torch.full((N,), 1e-3, device="cuda")
    step = torch.tensor(1.0, device="cuda")

    def adam(pp, gg, mm, vv):
        torch._fused_adam_([pp], [gg], [mm], [vv], [], [step], amsgrad=False, lr=1e-3, beta1=0.9, beta2=0.999,
                           weight_decay=0.0, eps=1e-8, maximize=False)

    def ar_then_adam():
        dist.all_reduce(gt)
        adam(pt, gt, mt, vt)

    _try(res, "nccl_allreduce_plus_torch_fused_adam_us", lambda: dtime(ar_then_adam, steps=50) * 1e3)
    sh = N // W
    gs, ps_, ms_, vs_ = (torch.zeros(sh, device="cuda") for _ in range(4))

    def rs_adam_ag():
        dist.reduce_scatter_tensor(gs, gt)
        adam(ps_, gs, ms_, vs_)
        dist.all_gather_into_tensor(pt, ps_)

    _try(res, "nccl_rs_torch_fused_adam_ag_us", lambda: dtime(rs_adam_ag, steps=50) * 1e3)
    best = [res[k] for k in ("nccl_allreduce_plus_torch_fused_adam_us", "nccl_rs_torch_fused_adam_ag_us")
            if isinstance(res.get(k), float)]
    if best:
        res["speedup_vs_best_nccl_baseline"] = min(best) / min(res["fused_fast_two_shot_us"],
                                                                res["fused_fast_one_shot_us"])
    out["c1"] = res
    for b in (g, p, m, v):
        ctx.free(b)
    tl.close()


def c3(ctx, out, nvl_peak, tc_peak):
    W, rows, H = ctx.world, 8192, 3072
    if H % (W * 64) and W > 1:
        out["c3"] = {"skipped": f"K = {H}/{W} is not a multiple of 64"}
        return
    k = H // W
    dt = torch.bfloat16
    x, w = ctx.alloc([rows, k], dt), ctx.alloc([k, H], dt)
    part, bb, rr, o1 = ctx.alloc([rows, H], dt), ctx.alloc([H], dt), ctx.alloc([rows, H], dt), ctx.alloc([rows, H], dt)
    ctx.view(x).normal_()
    ctx.view(w).normal_(0, k ** -0.5)
    ctx.view(bb).normal_(0, 0.1)
    ctx.view(rr).normal_()
    hp = BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_FAST)
    nvl = 2 * (W - 1) / W * rows * H * 2
    flops = 2.0 * rows * H * k
    res = {"workload": f"MP [8192x{k}]x[{k}x3072] bf16 + RS-bias-dropout-residual-AG, W={W}",
           "nvlink_bytes_per_rank_dir": nvl, "gemm_flops_per_rank": flops}
    f = lambda: mm_overlap_fused_ar(ctx, x, w, bb, rr, part, o1, hp)  # noqa: E731
    # AUTO: the all-gather -> GEMM kernel where cols/W is 128/256/384 (W=8 at
    # C3), else GEMM then the fused all-reduce
    res["auto_us"] = dtime(f) * 1e3
    for name, env in (("sequential_us", "sequential"), ("one_kernel_overlap_us", "fused")):
        os.environ["COCONET_MP_OVERLAP"] = env
        try:
            res[name] = dtime(f) * 1e3
        finally:
            os.environ.pop("COCONET_MP_OVERLAP", None)
    ctx.check()
    best = min(res["auto_us"], res["sequential_us"], res["one_kernel_overlap_us"])
    target_s = max(flops / (tc_peak * 1e12), nvl / (nvl_peak * 1e9))
    res["roofline_frac"] = target_s / (best * 1e-6)
    xt, wt = ctx.view(x).clone(), ctx.view(w).clone()
    bt, rt = ctx.view(bb).clone(), ctx.view(rr).clone()

    def baseline():
        y = xt @ wt
        dist.all_reduce(y)
        torch.nn.functional.dropout(y + bt, 0.1, training=True).add_(rt)

    _try(res, "nccl_matmul_allreduce_epilogue_us", lambda: dtime(baseline) * 1e3)
    if isinstance(res.get("nccl_matmul_allreduce_epilogue_us"), float):
        res["speedup_vs_nccl_baseline"] = res["nccl_matmul_allreduce_epilogue_us"] / best
    out["c3"] = res
    for b in (x, w, part, bb, rr, o1):
        ctx.free(b)


def c4(ctx, out, nvl_peak):
    W = ctx.world
    if W % 2:
        out["c4"] = {"skipped": "needs an even number of ranks (2 stages)"}
        return
    S, N, r = W // 2, C4_N, ctx.rank
    g0, g1 = ctx.group(0, S), ctx.group(S, S)
    res = {"workload": f"PP boundary 2x{S}, N={N}"}
    stage_pg = [dist.new_group(list(range(0, S))), dist.new_group(list(range(S, W)))]
    for dt, dn in ((torch.float16, "fp16"), (torch.float32, "fp32")):
        x, bb, rr, o = (ctx.alloc([N], dt) for _ in range(4))
        for t in (x, bb, rr):
            ctx.view(t).uniform_(0.1, 0.9)
        bw = 2 if dt == torch.float16 else 4
        nvl = N * bw  # per GPU per direction
        hp = BdrHParams(0.1, 1, 3251584743947114031, _lib.MATH_FAST)
        ms = dtime(lambda: rs_fused_send_ag(ctx, g0, g1, x, bb, rr, o, hp))
        res[f"fused_{dn}_us"] = ms * 1e3
        res[f"fused_{dn}_nvlink_frac"] = nvl / (ms * 1e-3) / 1e9 / nvl_peak
        ctx.check()
        xt, bt, rt = ctx.view(x).clone(), ctx.view(bb).clone(), ctx.view(rr).clone()
        sl = torch.empty(N // S, dtype=dt, device="cuda")
        full = torch.empty(N, dtype=dt, device="cuda")
        me = r % S

        gloo = dist.get_backend() == "gloo"  # share mode: gloo's send/recv take host tensors only
        sl_host = torch.empty(N // S, dtype=dt) if gloo else None

        def baseline():
            if r < S:  # stage 0: all_reduce, epilogue, send the rank's slice to its peer in stage 1
                dist.all_reduce(xt, group=stage_pg[0])
                y = torch.nn.functional.dropout(xt + bt, 0.1, training=True).add_(rt)
                piece = y[me * (N // S):(me + 1) * (N // S)].contiguous()
                dist.send(piece.cpu() if gloo else piece, dst=r + S)
            else:  # stage 1: receive the slice, all_gather the stage's slices
                if gloo:
                    dist.recv(sl_host, src=r - S)
                    sl.copy_(sl_host)
                else:
                    dist.recv(sl, src=r - S)
                dist.all_gather_into_tensor(full, sl, group=stage_pg[1])

        _try(res, f"nccl_ar_epilogue_send_ag_{dn}_us", lambda: dtime(baseline) * 1e3)
        if isinstance(res.get(f"nccl_ar_epilogue_send_ag_{dn}_us"), float):
            res[f"speedup_vs_nccl_baseline_{dn}"] = res[f"nccl_ar_epilogue_send_ag_{dn}_us"] / res[f"fused_{dn}_us"]
        for b in (x, bb, rr, o):
            ctx.free(b)
    out["c4"] = res


def c5(ctx, out, nvl_peak):
    W = ctx.world
    n = C5_PARAMS // (64 if share_mode() else 1)
    tl = TensorList(ctx, [n], bucket_cap=16384)
    g, p = ctx.alloc([n]), ctx.alloc([n])
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    ctx.view(g).normal_()
    ctx.view(p).uniform_(0.1, 0.9)
    ctx.view(m).zero_()
    ctx.view(v).fill_(1e-3)
    nvl = 2 * (W - 1) / W * n * 4
    res = {"workload": f"Adam {n} fp32 params, W={W}" + (" (scaled /64: share mode)" if share_mode() else ""),
           "nvlink_bytes_per_rank_dir": nvl}
    hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, _lib.MATH_FAST, _lib.ALGO_TWO_SHOT)
    ms = dtime(lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp), steps=3, warmup=2)
    ctx.check()
    res["fused_ms"] = ms
    res["fused_nvlink_frac"] = nvl / (ms * 1e-3) / 1e9 / nvl_peak
    for b in (m, v):
        ctx.free(b)
    # NCCL all_reduce + torch._fused_adam_ over the full (replicated) state, in 2^30 chunks
    try:
        gt = ctx.view(g)
        pt = ctx.view(p)
        mt = torch.zeros(n, device="cuda")
        vt = torch.full((n,), 1e-3, device="cuda")
        ch = 1 << 30
        parts = [(pt[i:i + ch], gt[i:i + ch], mt[i:i + ch], vt[i:i + ch]) for i in range(0, n, ch)]
        steps = [torch.tensor(1.0, device="cuda") for _ in parts]

        def baseline():
            dist.all_reduce(gt)
            torch._fused_adam_([a for a, _, _, _ in parts], [b for _, b, _, _ in parts],
                               [c for _, _, c, _ in parts], [d for _, _, _, d in parts], [], steps, amsgrad=False,
                               lr=1e-3, beta1=0.9, beta2=0.999, weight_decay=0.0, eps=1e-8, maximize=False)

        res["nccl_allreduce_plus_torch_fused_adam_ms"] = dtime(baseline, steps=3, warmup=2)
        res["speedup_vs_nccl_baseline"] = res["nccl_allreduce_plus_torch_fused_adam_ms"] / ms
        del mt, vt, parts
    except Exception as e:
        res["nccl_allreduce_plus_torch_fused_adam_ms"] = {"failed": repr(e)[:300]}
    torch.cuda.empty_cache()
    for b in (g, p):
        ctx.free(b)
    tl.close()
    out["c5"] = res


def _max_rel_dev(a, b) -> float:
    """max |a - b| over the largest magnitude of either (the tests' measure), on the device."""
    a, b = torch.as_tensor(a).double().flatten(), torch.as_tensor(b).double().flatten()
    if a.numel() == 0:
        return 0.0
    scale = max(1e-12, float(a.abs().max()), float(b.abs().max()))
    return float((a - b).abs().max()) / scale


def nvls(ctx, out, nvl_peak):
    """NVLS (NVSwitch multicast) against the P2P two-shot on the same inputs:
    fused Adam (C1 size and 2^26), the tensor-list AllReduce (2^26 fp32) and
    fused LAMB on the BERT-336M list (fp16 g). Runs only when every rank can
    create a multicast object (coconet_nvls_supported); the setup fails on all
    ranks together (runtime.Context._nvls_setup). Reported beside two-shot:
    time, and the max relative deviation from two-shot's result after one
    call from identical state (the switch sums in its own order)."""
    from paper_2105_05720_b200.collectives import LambHParams, allreduce, fused_rs_lamb_ag
    from paper_2105_05720_b200.runtime import Context, nvls_supported
    from paper_2105_05720_b200.workloads import bert_large_counts

    W, r = ctx.world, ctx.rank
    ok, why = nvls_supported(ctx.device, W)
    if share_mode() or max_over(0.0 if ok else 1.0) > 0:
        out["nvls"] = {"unavailable": why or "multicast unsupported on another rank (or share mode)"}
        return
    counts = bert_large_counts()
    n_l = sum(counts)
    heap = 2 * (n_l * 6 + 2 * (n_l // W + (1 << 20)) * 4) + (3 << 30)
    nctx = Context(W, mode="distributed", rank=r, device=ctx.device, heap_bytes=heap, heap="nvls")
    res = {"workload": f"W={W}: Adam fp32 2^20 / 2^26, AllReduce fp32 2^26, LAMB BERT-336M fp16 g",
           "mode": "NVLS: multimem.ld_reduce RS + multimem.st AG through the NVSwitch",
           "p2p_two_shot_nvlink_bytes_per_rank_dir_per_elem_fp32": 2 * (W - 1) / W * 4,
           "nvls_nvlink_bytes_per_rank_dir_per_elem_fp32": (W + 1) / W * 4}
    try:
        for n in (1 << 20, 1 << 26):
            tl = TensorList(nctx, [n])
            g, p = nctx.alloc([n]), nctx.alloc([n])
            m, v = nctx.alloc([tl.state_elems]), nctx.alloc([tl.state_elems])
            got = {}
            for algo, an in ((_lib.ALGO_TWO_SHOT, "two_shot"), (_lib.ALGO_NVLS, "nvls")):
                def reset():
                    torch.manual_seed(r)
                    nctx.view(g).normal_()
                    torch.manual_seed(100)
                    nctx.view(p).uniform_(0.1, 0.9)
                    nctx.view(m).zero_()
                    nctx.view(v).fill_(1e-3)
                    torch.cuda.synchronize()
                    dist.barrier()
                hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, _lib.MATH_FAST, algo)
                reset()
                fused_rs_adam_ag(nctx, tl, [g], [p], m, v, hp)
                nctx.check()
                got[an] = nctx.view(p).clone()
                res[f"adam_{n}_{an}_us"] = dtime(lambda: fused_rs_adam_ag(nctx, tl, [g], [p], m, v, hp),
                                                 steps=20) * 1e3
            res[f"adam_{n}_nvls_max_rel_dev"] = max_over(_max_rel_dev(got["nvls"], got["two_shot"]))
            res[f"adam_{n}_nvls_speedup"] = res[f"adam_{n}_two_shot_us"] / res[f"adam_{n}_nvls_us"]
            if n == 1 << 26:
                o = nctx.alloc([n])
                outs = {}
                for algo, an in ((_lib.ALGO_TWO_SHOT, "two_shot"), (_lib.ALGO_NVLS, "nvls")):
                    allreduce(nctx, tl, [g], [o], algo=algo)
                    nctx.check()
                    outs[an] = nctx.view(o).clone()
                    res[f"allreduce_{n}_{an}_us"] = dtime(lambda: allreduce(nctx, tl, [g], [o], algo=algo),
                                                          steps=20) * 1e3
                res[f"allreduce_{n}_nvls_max_rel_dev"] = max_over(_max_rel_dev(
                    outs["nvls"], outs["two_shot"]))
                res[f"allreduce_{n}_nvls_speedup"] = res[f"allreduce_{n}_two_shot_us"] / res[f"allreduce_{n}_nvls_us"]
                nctx.free(o)
            for b in (g, p, m, v):
                nctx.free(b)
            tl.close()
        # LAMB, BERT-336M list, fp16 g: the default schedule across ranks (TMA) vs NVLS
        tl = TensorList(nctx, counts, bucket_cap=16384)
        gs = [nctx.alloc([n], torch.float16) for n in counts]
        ps = [nctx.alloc([n]) for n in counts]
        m, v = nctx.alloc([tl.shard_elems]), nctx.alloc([tl.shard_elems])
        got = {}
        for sched, sn in ((_lib.LAMB_AUTO, "auto"), (_lib.LAMB_NVLS, "nvls")):
            torch.manual_seed(r)
            for x in gs:
                nctx.view(x).normal_()
            torch.manual_seed(100)
            for x in ps:
                nctx.view(x).uniform_(0.1, 0.9)
            nctx.view(m).zero_()
            nctx.view(v).fill_(1e-3)
            torch.cuda.synchronize()
            dist.barrier()
            hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched)
            fused_rs_lamb_ag(nctx, tl, gs, ps, m, v, hp)
            nctx.check()
            got[sn] = torch.cat([nctx.view(x) for x in ps])
            res[f"lamb_bert_{sn}_ms"] = dtime(lambda: fused_rs_lamb_ag(nctx, tl, gs, ps, m, v, hp), steps=10)
        res["lamb_bert_nvls_max_rel_dev"] = max_over(_max_rel_dev(got["nvls"], got["auto"]))
        res["lamb_bert_nvls_speedup"] = res["lamb_bert_auto_ms"] / res["lamb_bert_nvls_ms"]
        tl.close()
    finally:
        out["nvls"] = res
        torch.cuda.synchronize()
        dist.barrier()
        nctx.close()


def run_all(ctx, nvl_peak, tc_peak, only=("c1", "c3", "c4", "c5", "nvls")):
    """Runs the configs (collective). Returns the dict rank 0 reports."""
    out = {"mode": "DISTRIBUTED, one process per GPU" + (" (share mode: all ranks on GPU 0, gloo)" if share_mode()
                                                           else ", peers over NVLink, NCCL for the baselines"),
           "nvlink_peak_gbs": nvl_peak}
    for name in only:
        fn = {"c1": lambda: c1(ctx, out, nvl_peak), "c3": lambda: c3(ctx, out, nvl_peak, tc_peak),
              "c4": lambda: c4(ctx, out, nvl_peak), "c5": lambda: c5(ctx, out, nvl_peak),
              "nvls": lambda: nvls(ctx, out, nvl_peak)}[name]
        try:
            fn()
        except Exception as e:
            traceback.print_exc(file=sys.stderr)
            out[name] = {"failed": repr(e)[:300]}
        torch.cuda.synchronize()
        dist.barrier()
    return out


def main():
    """Standalone: torchrun --nproc-per-node N tools/dist_extras.py [c1,c3,...]"""
    import json

    from paper_2105_05720_b200.runtime import Context

    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    local = 0 if share_mode() else int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if share_mode():
        dist.init_process_group("gloo")
    else:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    only = tuple(sys.argv[1].split(",")) if len(sys.argv) > 1 else ("c1", "c3", "c4", "c5", "nvls")
    n5 = C5_PARAMS // (64 if share_mode() else 1)
    ctx = Context(world, mode="distributed", rank=rank, device=local,
                  heap_bytes=2 * n5 * 4 + 2 * (n5 // world + (1 << 20)) * 4 + (2 << 30))
    out = run_all(ctx, 770.0, 1634.5, only)
    if rank == 0:
        print(json.dumps(out))
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
