#!/usr/bin/env python
"""Benchmark of the fused data-parallel optimizer step (BASELINE.json metric:
"fused AR+Adam/LAMB step time & NVLink-roofline fraction, 1/2/4/8 B200").

Workload (BASELINE.json configs[1]): the BERT-large 336M gradient set — 398
tensors, 336,232,258 elements — as a tensor list (no flatten), fp16 gradients,
fp32 master weights and LAMB state; one step = ONE fused
ReduceScatter + LAMB + AllGather launch over the whole list. Synthetic values
are generated on the device (gen_decl_values semantics). The per-step traffic
(~13 GB at N=1) is 100x the 126 MB L2, so no L2 flush is needed between steps.

N=1: one GPU (one rank). N>1: torchrun, one process per GPU, peers mapped
over NVLink (DISTRIBUTED mode), weak scaling (every rank holds a full gradient
set, as in data parallelism). value = gradient elements reduced and applied
per second over the whole job = N * 336,232,258 / step time.

--impl reference times the reference's own CPU implementation (the UNMODIFIED
ccopt Engine compiled in place, oracle/_ref) on the same workload definition:
the authored LAMB fused program (tests/golden/lamb_fused_program.json) over a
bounded sample, on every host core (one Engine per core).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

METRIC = "fused AR+Adam/LAMB step time & NVLink-roofline fraction, 1/2/4/8 B200"
UNIT = "Gelem/s"
NVLINK_GBS = 770.0  # B200_PROFILING.md's measured peer copy per direction (900 nominal); at N>1
# bench.py measures its own peer copy and uses that when it can
BUCKET_CAP = 16384  # N=1: segments of the TMA LAMB schedule
BUCKET_CAP_MULTI = 16384  # N>1: the TMA schedule across ranks is fastest at 16384
# (W=2/8 virtual, profiles/r01_lamb_w_probe.json); GRID would prefer 4096
E2E_GROUPS = int(os.environ.get("COCONET_E2E_GROUPS", "16"))  # tensor groups pipelined against PCIe (e2e)
CPU_SAMPLE = 10 << 20  # elements per core for cpu_baseline: ~15 s of CPU work on the B200 host (4M took 6 s)


def peaks():
    """Roofline denominators: the driver-measured HBM copy GB/s and burst bf16
    TFLOP/s (MEASURED_PEAKS.json), else B200_PROFILING.md's fallback."""
    p = ROOT / "MEASURED_PEAKS.json"

    def num(x):
        if isinstance(x, dict):  # tolerate {"value": ...} entries
            x = x.get("value", x.get("median"))
        return float(x)

    if p.exists():
        try:
            d = json.loads(p.read_text())
            return num(d["hbm_gbs"]), num(d["bf16_tflops"]), "measured"
        except (KeyError, TypeError, ValueError) as e:
            print(f"bench: MEASURED_PEAKS.json unreadable ({e!r}); using the fallback peaks", file=sys.stderr)
    return 6650.0, 1590.0, "fallback"


# ---------------------------------------------------------------------------
# clocks sampled during the timed region (B200_PROFILING.md recipe)

class ClockSampler:
    """Polls NVML every 10 ms during the timed region: SM clock and the
    throttle reasons the recipe rejects on (B200_PROFILING.md)."""

    REASONS = {"hw_slowdown": 0x8, "sw_thermal_slowdown": 0x20, "hw_thermal_slowdown": 0x40,
               "sw_power_cap": 0x4}

    def __init__(self, device: int):
        self.device = device
        self.samples = []
        self.stop_flag = threading.Event()
        self.thread = None
        self.max_mhz = None
        self.error = None

    def start(self):
        self.error = None
        try:
            import pynvml
            pynvml.nvmlInit()
            # NVML numbers GPUs ignoring CUDA_VISIBLE_DEVICES: resolve the
            # handle of THIS CUDA device by its PCI bus id
            h = None
            try:
                import torch
                bus = torch.cuda.get_device_properties(self.device).pci_bus_id
                if bus:
                    h = pynvml.nvmlDeviceGetHandleByPciBusId_v2(bus.encode() if isinstance(bus, str) else bus)
            except Exception:
                h = None
            if h is None:
                h = pynvml.nvmlDeviceGetHandleByIndex(self.device)
            self.max_mhz = float(pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM))
            reasons_fn = getattr(pynvml, "nvmlDeviceGetCurrentClocksEventReasons", None) or \
                getattr(pynvml, "nvmlDeviceGetCurrentClocksThrottleReasons")
        except Exception as e:
            self.error = repr(e)
            return

        def run():
            while not self.stop_flag.is_set():
                try:
                    mhz = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
                    self.samples.append((float(mhz), int(reasons_fn(h))))
                except Exception as e:
                    self.error = repr(e)
                time.sleep(0.01)

        self.thread = threading.Thread(target=run, daemon=True)
        self.thread.start()

    def stop(self):
        self.stop_flag.set()
        if self.thread:
            self.thread.join(timeout=1)
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "samples": 0, "reasons": ["unsampled"],
                    "sampling_error": self.error}
        active = sorted({n for _, bits in self.samples for n, m in self.REASONS.items() if bits & m})
        return {"sm_mhz": statistics.median(m for m, _ in self.samples), "sm_max_mhz": self.max_mhz,
                "samples": len(self.samples), "reasons": active, "source": "NVML, 10 ms"}


# ---------------------------------------------------------------------------
# reference CPU path (oracle/_ref): the reference Engine on the LAMB program

def reference_cpu(sample_elems: int, threads: int, steps: int = 1):
    """Runs `threads` independent reference Engines concurrently (one per host
    core; the reference's own Threaded mode only spawns one thread per rank,
    runtime.hpp:287-296, i.e. one thread at W=1), each on an N=sample_elems
    instance of the authored fused LAMB program at W=1. Returns (elem/s, wall)."""
    from oracle import ref

    base = (ROOT / "tests" / "golden" / "lamb_program.json").read_text()
    fused = (ROOT / "tests" / "golden" / "lamb_fused_program.json").read_text()
    sessions = []
    for i in range(threads):
        s = ref.RefSession(base, None, {"N": sample_elems, "W": 1}, sched_program=fused)
        s.gen(1 + i)
        sessions.append(s)
    times = [0.0] * threads

    def work(i):
        t = 0.0
        for _ in range(steps):
            t += sessions[i].time_engine(1 + i, ref.ENGINE_SCHED)
        times[i] = t

    t0 = time.perf_counter()
    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - t0
    return threads * steps * sample_elems / wall, wall


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    from oracle import ref

    if not ref.available():
        print(json.dumps({"impl": "reference", "metric": METRIC,
                          "unavailable": "oracle/_ref/libccopt_ref.so not built (needs /root/reference at build time)"}))
        return
    cores = os.cpu_count() or 1
    sample = 1 << 21  # per core per step: ~3-4 s of CPU work on 16 cores
    # warmup steps, then timed steps; each step is a bounded sample per core
    for _ in range(max(0, min(args.warmup, 1))):
        reference_cpu(sample, cores, 1)
    rate, wall = reference_cpu(sample, cores, args.steps)
    value = rate / 1e9
    from paper_2105_05720_b200.workloads import BERT_LARGE_PARAMS
    ms = BERT_LARGE_PARAMS / rate * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (gen_decl_values, seed per core)",
        "config": {"workload": "BERT-336M LAMB step (398 tensors, 336,232,258 params), "
                               "reference Engine on tests/golden/lamb_fused_program.json",
                   "sample": f"{cores} concurrent Engines x N={sample} elements x {args.steps} steps, W=1",
                   "ms_per_step_is": "extrapolated to 336,232,258 elements at the measured rate"},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "reference",
                         "sample": f"{cores} x {sample} elements x {args.steps} steps in {wall:.1f} s"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line))


# ---------------------------------------------------------------------------
# the CUDA path

def lamb_parity(ctx, tl, counts, grads, params, m, v, hp, world, rank, distributed):
    """One fused step after the timed region, checked against an fp64 torch
    evaluation of the LAMB definition (tests/golden/lamb_list_*: per tensor
    m' = b1 m + (1-b1) g, v' = b2 v + (1-b2) g^2, u = m'/bc1 / (sqrt(v'/bc2) +
    eps) + wd p, p' = p - lr ||p||/||u|| u) on the pre-step state, over EVERY
    tensor: p (this rank's gathered copy), m and v (every rank's shard). g is
    the sum of all ranks' fp16 gradients. Tolerance: the north star's 1e-5
    for fp32 optimizer state."""
    import math

    import torch
    import torch.distributed as dist

    me = ctx.local_ranks()[0]
    dev = torch.device("cuda")

    def shards(buf):
        loc = ctx.view(buf, me).clone()
        if not distributed:
            return [loc]
        allb = [torch.empty_like(loc) for _ in range(world)]
        dist.all_gather(allb, loc)
        return allb

    m0, v0 = shards(m), shards(v)
    p0 = [ctx.view(b, me).clone() for b in params]
    g_sum = []
    for b in grads:
        x = ctx.view(b, me).double()
        if distributed:
            dist.all_reduce(x)
        g_sum.append(x)
    fused_rs_lamb_ag = __import__("paper_2105_05720_b200.collectives", fromlist=["x"]).fused_rs_lamb_ag
    fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
    ctx.check()
    m1, v1 = shards(m), shards(v)
    # element -> shard position per tensor, from every rank's segment table
    idx = [[] for _ in counts]
    for r in range(world):
        segs = torch.from_numpy(tl.segments(r))
        for t, toff, ln, sidx in segs.tolist():
            idx[t].append((toff, ln, r, sidx))
    b1, b2 = float(hp.beta1), float(hp.beta2)
    bc1, bc2 = 1 - b1 ** hp.t, 1 - b2 ** hp.t
    worst, checked = 0.0, 0
    for t, n in enumerate(counts):
        pos = torch.empty(n, dtype=torch.int64)
        src = torch.empty(n, dtype=torch.int64)
        for toff, ln, r, sidx in idx[t]:
            pos[toff:toff + ln] = torch.arange(sidx, sidx + ln)
            src[toff:toff + ln] = r
        pos, src = pos.to(dev), src.to(dev)
        stack = lambda parts: torch.stack(parts)[src, pos]  # noqa: E731
        mo, vo = stack(m0).double(), stack(v0).double()
        g, p = g_sum[t], p0[t].double()
        mn = b1 * mo + (1 - b1) * g
        vn = b2 * vo + (1 - b2) * g * g
        u = (mn / bc1) / ((vn / bc2).sqrt() + float(hp.eps)) + float(hp.wd) * p
        pn = p - float(hp.lr) * math.sqrt(float((p * p).sum())) / math.sqrt(float((u * u).sum())) * u

        def dev_of(a, b):
            return float((a.double() - b).abs().max() / torch.maximum(a.double().abs().max(), b.abs().max()).clamp_min(1e-12))

        worst = max(worst, dev_of(ctx.view(params[t], me), pn), dev_of(stack(m1), mn), dev_of(stack(v1), vn))
        checked += 1
    if distributed:
        from paper_2105_05720_b200.runtime import max_over_ranks
        worst = max_over_ranks(worst)
    return {"max_rel_dev": worst, "tensors_checked": checked, "tolerance": 1e-5, "ok": worst <= 1e-5,
            "checker": "torch fp64 LAMB definition on the pre-step state (p, m, v of every tensor)"}


def run_coconet(args):
    import torch
    import torch.distributed as dist

    from paper_2105_05720_b200 import _lib  # noqa: F401
    from paper_2105_05720_b200.collectives import (AdamHParams, LambHParams, TensorList, fused_rs_adam_ag,
                                                   fused_rs_lamb_ag, gen_values, unfused_lamb)
    from paper_2105_05720_b200.runtime import Context, max_over_ranks
    from paper_2105_05720_b200.workloads import BERT_LARGE_PARAMS, bert_large_counts

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    # test-only: run every rank on GPU 0 (CUDA IPC works between processes on
    # one device; NCCL does not accept duplicate GPUs, so bootstrap over gloo)
    share = os.environ.get("COCONET_SHARE_DEVICE") == "1"
    if share:
        local_rank = 0
    assert world == args.gpus, f"--gpus {args.gpus} but WORLD_SIZE={world}"
    torch.cuda.set_device(local_rank)
    distributed = world > 1
    if distributed:
        if share:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    counts = bert_large_counts()
    padded = [(n + 63) // 64 * 64 for n in counts]
    W = world
    shard_state = 2 * (sum(counts) // W + 64 * len(counts) + 4096) * 4  # m + v of one rank's shard
    full_state = (sum(counts) + 64 * len(counts) + 4096) * 4  # one fp32 buffer over the size-1 group's list
    need = (sum(padded) * (2 + 4) + shard_state  # flat g, p + the fused step's m, v
            + shard_state + 2 * 8192 * E2E_GROUPS * 4  # the e2e pipeline's per-group m, v
            + 3 * full_state  # the unfused baseline's replicated m, v and its u scratch
            + (256 << 20))
    ctx = Context(W, mode="distributed" if distributed else "virtual", rank=rank, device=local_rank,
                  heap_bytes=need)
    # bucket capacity: the reference's 2^10 (runtime.hpp:579) fixes the flat order
    # the parity tests pin; for this workload 16384-element buckets amortise the
    # per-segment cost of the TMA ring (descriptor + per-segment norm), DESIGN.md §3
    cap = BUCKET_CAP if world == 1 else BUCKET_CAP_MULTI
    tl = TensorList(ctx, counts, bucket_cap=cap)
    # one flat buffer per dtype (tensors at 64-element aligned offsets) so the
    # unfused baseline can hand all gradients to ONE NCCL all_reduce
    from paper_2105_05720_b200.runtime import SymmBuffer
    flat_g = ctx.alloc([sum(padded)], torch.float16)
    flat_p = ctx.alloc([sum(padded)], torch.float32)
    grads, params, off = [], [], 0
    for n, pn in zip(counts, padded):
        grads.append(SymmBuffer(flat_g.offset + off * 2, (n,), torch.float16))
        params.append(SymmBuffer(flat_p.offset + off * 4, (n,), torch.float32))
        off += pn
    m = ctx.alloc([tl.shard_elems], torch.float32)
    v = ctx.alloc([tl.shard_elems], torch.float32)
    my_ranks = ctx.local_ranks()
    for r in my_ranks:
        for i, n in enumerate(counts):
            gen_values(ctx, ctx.view(grads[i], r), 1, f"g{i}", "local", r, [n], group_size=W)
            gen_values(ctx, ctx.view(params[i], r), 1, f"p{i}", "replicated", r, [n], group_size=W)
        ctx.view(m, r).uniform_(-1e-3, 1e-3)
        ctx.view(v, r).uniform_(1e-4, 1e-3)
    hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, eps=1e-6, wd=0.01)
    stream = torch.cuda.current_stream()
    torch.cuda.synchronize()

    def step():
        fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)

    def barrier():
        torch.cuda.synchronize()
        if distributed:
            dist.barrier()
        torch.cuda.synchronize()

    def event_time(fn, steps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        barrier()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        barrier()
        t = e0.elapsed_time(e1) / steps
        return max_over_ranks(t) if distributed else t

    for _ in range(args.warmup):
        step()
    ctx.check()
    barrier()

    def timed():
        sampler = ClockSampler(local_rank)
        sampler.start()
        launches0 = ctx.launch_count()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        torch.cuda.nvtx.range_push("timed")  # ncu --nvtx-include "timed/" captures exactly these launches
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.nvtx.range_pop()
        barrier()
        clocks = sampler.stop()
        ctx.check()
        t = e0.elapsed_time(e1) / args.steps
        return (max_over_ranks(t) if distributed else t), clocks, ctx.launch_count() - launches0

    ms, clocks, launches = timed()
    # the recipe's rejection rule: a slowdown reason, or SM clocks well below
    # max with no reason (a leftover lock), re-measures once (on every rank)
    bad = bool(set(clocks["reasons"]) & {"hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown"}) or (
        clocks["sm_mhz"] is not None and clocks["sm_max_mhz"] and not clocks["reasons"]
        and clocks["sm_mhz"] < 0.85 * clocks["sm_max_mhz"])
    if (max_over_ranks(float(bad)) if distributed else float(bad)) > 0:
        first = clocks
        ms, clocks, launches = timed()
        clocks = dict(clocks, remeasured_after=first)
    N = BERT_LARGE_PARAMS
    value = W * N / (ms * 1e-3) / 1e9

    # -- parity of the timed call: one more step, every tensor checked
    parity = None
    if not args.no_parity:
        try:
            parity = lamb_parity(ctx, tl, counts, grads, params, m, v, hp, world, rank, distributed)
        except Exception as e:
            parity = {"failed": repr(e)[:300]}
        torch.cuda.empty_cache()

    # -- the unfused GPU baseline (north star: "NCCL plus separate kernels"):
    # NCCL all_reduce of the flat fp16 gradients (N > 1), then the same LAMB
    # as apex FusedLAMB's FOUR separate multi-tensor kernels over all elements
    # on every rank (replicated state; coconet_unfused_lamb, csrc/unfused.cu)
    baseline = None
    if not args.no_baseline:
        try:
            g1 = ctx.group(ctx.local_ranks()[0], 1)
            tl1 = TensorList(ctx, counts, group=g1, bucket_cap=BUCKET_CAP)
            m1, v1, u1 = (ctx.alloc([tl1.shard_elems], torch.float32) for _ in range(3))
            ctx.view(m1).zero_() if distributed else ctx.view(m1, 0).zero_()
            (ctx.view(v1) if distributed else ctx.view(v1, 0)).fill_(1e-4)
            norms = torch.zeros(2 * len(counts), dtype=torch.float64, device="cuda")
            flat = ctx.view(flat_g) if distributed else ctx.view(flat_g, 0)

            def base_step():
                if distributed:
                    dist.all_reduce(flat)
                unfused_lamb(ctx, tl1, grads, params, m1, v1, u1, norms, hp)

            for _ in range(3):
                base_step()
            ctx.check()
            bms = event_time(base_step, max(3, min(args.steps, 10)))
            baseline = {"ms_per_step": bms, "value": W * N / (bms * 1e-3) / 1e9, "unit": UNIT,
                        "what": ("NCCL all_reduce (fp16, flat) + " if distributed else "") +
                                "apex-FusedLAMB-structured separate kernels (stage 1, l2norm partials, "
                                "per-tensor combine, stage 2: 46 B/element) over all elements per rank",
                        "fused_speedup": bms / ms}
            if distributed:
                baseline["nccl_allreduce_ms"] = event_time(lambda: dist.all_reduce(flat), 3)
            tl1.close()
            for b in (m1, v1, u1):
                ctx.free(b)
        except Exception as e:
            baseline = {"failed": repr(e)[:300]}
        if world == 1:  # Adam on the same list: the fused FAST kernel vs torch._fused_adam_ (fp32 grads)
            try:
                baseline["adam"] = adam_vs_torch(ctx, counts, event_time)
            except Exception as e:
                baseline["adam"] = {"failed": repr(e)[:300]}
        torch.cuda.empty_cache()

    # -- e2e: through the public API with HOST buffers (pinned): every step
    # copies this rank's fp16 gradients H2D and its updated fp32 parameters
    # D2H inside the timed region. LambHostPipeline overlaps the PCIe copies
    # with the fused launches by tensor groups (H2D(k+1) || LAMB(k) || D2H(k-1))
    from paper_2105_05720_b200.collectives import LambHostPipeline
    offsets = [0]
    for pn in padded[:-1]:
        offsets.append(offsets[-1] + pn)
    pipe = LambHostPipeline(ctx, counts, flat_g, flat_p, offsets, groups=E2E_GROUPS, bucket_cap=cap)
    for (pm, pv) in pipe.state():
        ctx.view(pm).uniform_(-1e-3, 1e-3)
        ctx.view(pv).uniform_(1e-4, 1e-3)
    me = my_ranks[0]
    h_g = ctx.view(flat_g, me).cpu().pin_memory()
    h_p = torch.empty(sum(padded), dtype=torch.float32).pin_memory()
    for _ in range(2):  # warm-up
        pipe.step(h_g, h_p, hp)
        pipe.wait()
    barrier()
    e2e_steps = max(3, min(args.steps, 10))
    t0 = time.perf_counter()
    for _ in range(e2e_steps):
        pipe.step(h_g, h_p, hp)
        pipe.wait()
    barrier()
    e2e_s = (time.perf_counter() - t0) / e2e_steps
    if distributed:
        e2e_s = max_over_ranks(e2e_s)
    h2d = pipe.h2d_bytes
    d2h = pipe.d2h_bytes

    # -- roofline of the dominant (only) kernel
    hbm_peak, tc_peak, peak_kind = peaks()
    nvl_peak, nvl_kind = NVLINK_GBS, "B200_PROFILING.md measured peer copy per direction (900 nominal)"
    if distributed and not share:
        try:
            from tools.dist_extras import peer_copy_gbs
            measured = max_over_ranks(-peer_copy_gbs(ctx))  # min over ranks
            nvl_peak, nvl_kind = -measured, "peer copy measured in this run (min over ranks, per direction)"
        except Exception:
            pass
    shard = N / W
    # per-rank HBM bytes: W=1 the ONCHIP schedule (AUTO) moves
    # 30 B/elem (pass 1: g 2 + m, v, p 12 read, m', v' 8 written; pass 2: p 4 +
    # 4) plus 8 B for every element whose u is not held on chip (past the hold,
    # or a per-window cover item; its pass 2
    # re-reads m', v'); the two-pass TMA schedule 38 B/elem. W>1 (TMA): the
    # shard's 38 B minus its g read / p write (served by the peers' HBM) plus
    # this rank's whole g read by its owners (2N) and whole p written by them (4N)
    spilled = tl.onchip_spilled() if W == 1 else -1
    sched_name = "ONCHIP" if spilled >= 0 else "TMA"
    if W == 1:
        hbm_bytes = 30.0 * shard + 8.0 * spilled if spilled >= 0 else 38.0 * shard
    else:
        hbm_bytes = 32.0 * shard + 6.0 * N
    nvl_bytes = (W - 1) / W * N * (2 + 4)
    if W == 1:
        achieved = hbm_bytes / (ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": hbm_bytes, "schedule": sched_name,
                "spilled_elems": spilled if spilled >= 0 else None,
                "compulsory_bytes_per_launch": 26.0 * N,
                "compulsory_frac": 26.0 * N / (ms * 1e-3) / 1e9 / hbm_peak}
    else:
        achieved = nvl_bytes / (ms * 1e-3) / 1e9
        roof = {"bound": "nvlink", "achieved": achieved, "peak": nvl_peak, "unit": "GB/s",
                "frac": achieved / nvl_peak, "peak_kind": nvl_kind,
                "algorithmic_bytes_per_launch": nvl_bytes,
                "hbm_bytes_per_launch": hbm_bytes, "hbm_frac": hbm_bytes / (ms * 1e-3) / 1e9 / hbm_peak}
    prof = ROOT / "profiles" / "ncu_traffic.json"
    roof["traffic"] = None
    if prof.exists() and W == 1:  # the committed capture is of the W=1 launch
        try:
            roof["traffic"] = json.loads(prof.read_text()).get("lamb_kernel", {}).get("dram_bytes_per_launch")
        except Exception:
            pass

    extras = None
    if not args.no_extras:
        if world == 1:
            # the other BASELINE configs on this GPU with virtual ranks (kernel and
            # protocol cost; "NVLink" traffic is local HBM here) - see DESIGN.md
            try:
                ctx.close()
                from tools.pattern_probe import c1, c2_w8, c3, c4, c5
                extras = {"note": "one GPU, virtual ranks: all ranks' traffic is local HBM"}
                for fn in (c1, c2_w8, c3, c4, c5):
                    fn(extras)
            except Exception as e:
                extras = {"failed": repr(e)}
        else:
            # the other BASELINE configs across the N GPUs, each beside its NCCL baseline
            try:
                ctx.close()  # a fresh symmetric heap sized for C5's 3.9e9 fp32 g and p
                from tools.dist_extras import C5_PARAMS, run_all
                n5 = C5_PARAMS // (64 if share else 1)
                ctx = Context(W, mode="distributed", rank=rank, device=local_rank,
                              heap_bytes=2 * n5 * 4 + 2 * (n5 // W + (1 << 20)) * 4 + (2 << 30))
                extras = run_all(ctx, nvl_peak, tc_peak)
            except Exception as e:
                extras = {"failed": repr(e)[:300]}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            from oracle import ref
            if ref.available():
                cores = os.cpu_count() or 1
                rate, wall = reference_cpu(CPU_SAMPLE, cores, 1)
                cpu = {"value": rate / 1e9, "unit": UNIT, "cores": cores, "kind": "reference",
                       "sample": f"{cores} concurrent reference Engines x {CPU_SAMPLE}-element LAMB "
                                 f"(tests/golden/lamb_fused_program.json, W=1) in {wall:.1f} s"}
        except Exception as e:  # the baseline is reported, not required
            cpu = {"value": None, "unit": UNIT, "cores": 0, "kind": "reference", "sample": f"failed: {e}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (device-generated, gen_decl_values semantics)",
            "config": {"workload": "BERT-336M LAMB step: 398-tensor list, 336,232,258 params, fp16 grads, "
                                   "fp32 master weights + m/v, fused ReduceScatter+LAMB+AllGather",
                       "global_batch": None, "seq_len": None, "parallelism": f"dp{world}",
                       "l2": "per-step traffic ~13 GB >> 126 MB L2 (no flush needed)",
                       "math": "FAST (fp32 element math, fp64 norms)", "bucket_cap": cap},
            "roofline": roof, "cpu_baseline": cpu,
            "e2e": {"value": W * N / e2e_s / 1e9, "unit": UNIT, "h2d_bytes_per_step": h2d,
                    "d2h_bytes_per_step": d2h,
                    "what": "pinned H2D of this rank's fp16 grads + fused step + D2H of updated fp32 params, "
                            f"pipelined by {len(pipe.groups)} tensor groups (collectives.LambHostPipeline)"},
            "gpu_launches": launches, "clocks": clocks,
            "kernel_ms": ms,
            "parity": parity,
            "unfused_baseline": baseline,
            "extras": extras,
        }
        print(json.dumps(line), flush=True)
    try:  # teardown after the line is out: a failure here must not cost the measurement
        if ctx.handle:
            ctx.close()
        if distributed:
            dist.destroy_process_group()
    except Exception as e:
        print(f"teardown: {e!r}", file=sys.stderr)


def adam_vs_torch(ctx, counts, event_time):
    """Adam over the BERT-336M list with fp32 grads: the fused FAST kernel
    (W=1: the TMA ring) vs torch._fused_adam_ (torch's own multi-tensor fused
    Adam) on the same tensors."""
    import torch

    from paper_2105_05720_b200.collectives import AdamHParams, TensorList, fused_rs_adam_ag

    g1 = ctx.group(ctx.local_ranks()[0], 1)
    tl = TensorList(ctx, counts, group=g1, bucket_cap=BUCKET_CAP)
    bufs_g = [ctx.alloc([n]) for n in counts]
    bufs_p = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    r = ctx.local_ranks()[0]
    for b in bufs_g:
        ctx.view(b, r).normal_()
    for b in bufs_p:
        ctx.view(b, r).uniform_(0.1, 0.9)
    ctx.view(m, r).zero_()
    ctx.view(v, r).fill_(1e-3)
    hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, 1, 1)  # FAST, TWO_SHOT
    fused = lambda: fused_rs_adam_ag(ctx, tl, bufs_g, bufs_p, m, v, hp)  # noqa: E731
    for _ in range(3):
        fused()
    ours = event_time(fused, 10)
    tp = [ctx.view(b, r) for b in bufs_p]
    tg = [ctx.view(b, r) for b in bufs_g]
    tm = [torch.zeros(n, device="cuda") for n in counts]
    tv = [torch.full((n,), 1e-3, device="cuda") for n in counts]
    steps = [torch.tensor(1.0, device="cuda") for _ in counts]
    ref = lambda: torch._fused_adam_(tp, tg, tm, tv, [], steps, amsgrad=False, lr=1e-3, beta1=0.9,  # noqa: E731
                                     beta2=0.999, weight_decay=0.0, eps=1e-8, maximize=False)
    for _ in range(3):
        ref()
    theirs = event_time(ref, 10)
    tl.close()
    for b in bufs_g + bufs_p + [m, v]:
        ctx.free(b)
    return {"fused_fast_ms": ours, "torch_fused_adam_ms": theirs, "fused_speedup": theirs / ours,
            "what": "Adam, BERT-336M list, fp32 grads/params/state, W=1"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="coconet", choices=["coconet", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-baseline", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_coconet(args)


if __name__ == "__main__":
    main()
