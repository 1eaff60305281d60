"""ONCHIP LAMB window-wait trace (profiling only, not the bench): the kernel
records, per window and CTA, when its pass 1 finished, when it reached the
pass-2 norm wait and when it was released (COCONET_LAMB_OC_TRACE = heap
offset of the trace buffer). BERT-336M list, W=1, fp16 g, 16384-element
buckets. Prints the per-window finish skew across CTAs, the wait each CTA
saw and the release latency after the last arrival.
The per-window fields belong to the per-window protocol (commit cf562ce);
since the per-tensor release only [2] (the window's last ratio ready in the
CTA) is recorded. Usage: python tools/lamb_trace_probe.py"""
import json
import os
import statistics
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import LambHParams, TensorList, fused_rs_lamb_ag, gen_values  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from paper_2105_05720_b200.workloads import bert_large_counts  # noqa: E402

MAXW, NG = 256, 148


def main():
    counts = bert_large_counts()
    N = sum(counts)
    ctx = Context(1, heap_bytes=N * 16 + (1 << 30))
    tl = TensorList(ctx, counts, bucket_cap=16384)
    grads = [ctx.alloc([n], torch.float16) for n in counts]
    params = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    for i, n in enumerate(counts):
        gen_values(ctx, ctx.view(grads[i], 0), 1, f"g{i}", "local", 0, [n], group_size=1)
        gen_values(ctx, ctx.view(params[i], 0), 1, f"p{i}", "replicated", 0, [n], group_size=1)
    ctx.view(m, 0).uniform_(-1e-3, 1e-3)
    ctx.view(v, 0).uniform_(1e-4, 1e-3)
    trace = ctx.alloc([MAXW * NG * 4], torch.int64)
    hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=_lib.LAMB_ONCHIP)
    for _ in range(3):
        fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
    ctx.view(trace, 0).zero_()
    torch.cuda.synchronize()
    os.environ["COCONET_LAMB_OC_TRACE"] = str(trace.offset)
    if len(sys.argv) > 1:  # e.g. 2: relaxed arrivals (profiling only)
        os.environ["COCONET_LAMB_OC_NOSYNC"] = sys.argv[1]
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
    e.record()
    torch.cuda.synchronize()
    os.environ.pop("COCONET_LAMB_OC_TRACE")
    os.environ.pop("COCONET_LAMB_OC_NOSYNC", None)
    ctx.check()
    t = ctx.view(trace, 0).view(MAXW, NG, 4).cpu()
    t0 = int(t[t > 0].min())
    windows = []
    for w in range(MAXW):
        fin, reach, rel = t[w, :, 0], t[w, :, 1], t[w, :, 2]
        if int(reach.max()) == 0:
            continue
        last = int(fin.max())
        waits = [(int(rel[c]) - int(reach[c])) / 1e3 for c in range(NG)]
        windows.append({
            "window": w,
            "finish_spread_us": (last - int(fin.min())) / 1e3,
            "finish_last_minus_median_us": (last - statistics.median(fin.tolist())) / 1e3,
            "wait_mean_us": statistics.mean(waits), "wait_max_us": max(waits),
            "release_after_last_arrival_us": (int(rel.min()) - last) / 1e3,
            "reach_before_last_arrival_frac": sum(1 for c in range(NG) if int(reach[c]) < last) / NG,
            "t_release_us": (int(rel.min()) - t0) / 1e3,
        })
    out = {"ms": s.elapsed_time(e), "windows": len(windows),
           "sum_of_mean_waits_us": sum(x["wait_mean_us"] for x in windows),
           "mean_finish_spread_us": statistics.mean(x["finish_spread_us"] for x in windows),
           "mean_release_latency_us": statistics.mean(x["release_after_last_arrival_us"] for x in windows),
           "per_window": windows}
    print(json.dumps({k: v for k, v in out.items() if k != "per_window"}, indent=1))
    for x in windows[:60]:
        print(x)
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/lamb_trace_probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
