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
NVLINK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md)
BUCKET_CAP = 16384  # N=1: segments of the TMA LAMB schedule
BUCKET_CAP_MULTI = 16384  # N>1: the TMA schedule across ranks is fastest at 16384
# (W=2/8 virtual, profiles/r01_lamb_w_probe.json); GRID would prefer 4096
E2E_GROUPS = 16  # tensor groups pipelined against PCIe in the e2e measurement
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

def run_coconet(args):
    import torch
    import torch.distributed as dist

    from paper_2105_05720_b200 import _lib
    from paper_2105_05720_b200.collectives import LambHParams, TensorList, fused_rs_lamb_ag, gen_values
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
    need = (sum(padded) * (2 + 4) + shard_state  # flat g, p + the fused step's m, v
            + shard_state + 2 * 8192 * E2E_GROUPS * 4  # the e2e pipeline's per-group m, v
            + (2 * sum(padded) * 4 if distributed else 0)  # the NCCL baseline's replicated m, v
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

    # -- the unfused GPU baseline (north star): NCCL all_reduce of the flat
    # fp16 gradients, then a separate LAMB over ALL elements on every rank
    # (replicated state, DDP + fused-optimizer style), on the same box
    nccl_baseline = None
    if distributed and not share:
        try:  # the baseline is reported, never allowed to sink the bench line
            g1 = ctx.group(rank, 1)
            tl1 = TensorList(ctx, counts, group=g1, bucket_cap=BUCKET_CAP)  # size-1 group: the TMA path
            m1 = ctx.alloc([tl1.shard_elems], torch.float32)
            v1 = ctx.alloc([tl1.shard_elems], torch.float32)
            ctx.view(m1).zero_()
            ctx.view(v1).fill_(1e-4)
            flat = ctx.view(flat_g)

            def base_step():
                dist.all_reduce(flat)
                fused_rs_lamb_ag(ctx, tl1, grads, params, m1, v1, hp)

            for _ in range(args.warmup):
                base_step()
            barrier()
            b0 = torch.cuda.Event(enable_timing=True)
            b1 = torch.cuda.Event(enable_timing=True)
            b0.record(stream)
            for _ in range(args.steps):
                base_step()
            b1.record(stream)
            barrier()
            bms = max_over_ranks(b0.elapsed_time(b1) / args.steps)
            nccl_baseline = {"ms_per_step": bms, "value": W * N / (bms * 1e-3) / 1e9, "unit": UNIT,
                             "what": "NCCL all_reduce (fp16, flat) + separate LAMB over all elements per rank",
                             "speedup_of_fused": bms / ms}
        except Exception as e:
            nccl_baseline = {"failed": repr(e)}

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
    shard = N / W
    # per-rank HBM bytes: W=1 two-pass LAMB = 38 B/elem; W>1 the
    # shard's 38 B minus its g read / p write (served by the peers' HBM) plus this
    # rank's whole g read by its owners (2N) and whole p written by them (4N)
    hbm_bytes = 38.0 * shard if W == 1 else 32.0 * shard + 6.0 * N
    nvl_bytes = (W - 1) / W * N * (2 + 4)
    if W == 1:
        achieved = hbm_bytes / (ms * 1e-3) / 1e9
        roof = {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                "frac": achieved / hbm_peak, "peak_kind": peak_kind,
                "algorithmic_bytes_per_launch": hbm_bytes}
    else:
        achieved = nvl_bytes / (ms * 1e-3) / 1e9
        roof = {"bound": "nvlink", "achieved": achieved, "peak": NVLINK_GBS, "unit": "GB/s",
                "frac": achieved / NVLINK_GBS, "peak_kind": "measured peer copy (B200_PROFILING.md)",
                "algorithmic_bytes_per_launch": nvl_bytes}
    prof = ROOT / "profiles" / "ncu_traffic.json"
    roof["traffic"] = None
    if prof.exists() and W == 1:  # the committed capture is of the W=1 launch
        try:
            roof["traffic"] = json.loads(prof.read_text()).get("lamb_kernel", {}).get("dram_bytes_per_launch")
        except Exception:
            pass

    extras = None
    if rank == 0 and world == 1 and not args.no_extras:
        # the other BASELINE configs on this GPU with virtual ranks (kernel and
        # protocol cost; "NVLink" traffic is local HBM here) - see DESIGN.md
        try:
            ctx.close()
            from tools.pattern_probe import c1, c2_w8, c3, c4, c5, unfused_baselines
            extras = {"note": "one GPU, virtual ranks: all ranks' traffic is local HBM"}
            for f in (c1, c2_w8, c3, c4, c5, unfused_baselines):
                f(extras)
            if "unfused_torch_foreach_lamb_bert336m_ms" in extras:
                extras["fused_lamb_speedup_vs_unfused"] = extras["unfused_torch_foreach_lamb_bert336m_ms"] / ms
        except Exception as e:
            extras = {"failed": repr(e)}

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
            "extras": extras,
            "nccl_baseline": nccl_baseline,
        }
        print(json.dumps(line))
    if ctx.handle:
        ctx.close()
    if distributed:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="coconet", choices=["coconet", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    if args.impl == "reference":
        run_reference(args)
    else:
        run_coconet(args)


if __name__ == "__main__":
    main()
