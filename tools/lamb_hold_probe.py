"""ONCHIP LAMB probe (not the bench): step time on the BERT-336M list (W=1,
fp16 g, 16384-element buckets) as the on-chip hold per CTA shrinks, with and
without the per-window norm wait (COCONET_LAMB_OC_NOSYNC=1 gives invalid
results: timing only). Measures what halving the window costs, the price of
holding p on chip next to u (the HP variant itself was measured and dropped:
profiles/r02_lamb_onchip_holdp.json). Usage: python tools/lamb_hold_probe.py"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import LambHParams, TensorList, fused_rs_lamb_ag, gen_values  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from paper_2105_05720_b200.workloads import bert_large_counts  # noqa: E402


def main():
    counts = bert_large_counts()
    N = sum(counts)
    ctx = Context(1, heap_bytes=N * 16 + (1 << 30))
    tl = TensorList(ctx, counts, bucket_cap=16384)
    grads = [ctx.alloc([n], torch.float16) for n in counts]
    params = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])

    def reset():
        for i, n in enumerate(counts):
            gen_values(ctx, ctx.view(grads[i], 0), 1, f"g{i}", "local", 0, [n], group_size=1)
            gen_values(ctx, ctx.view(params[i], 0), 1, f"p{i}", "replicated", 0, [n], group_size=1)
        ctx.view(m, 0).uniform_(-1e-3, 1e-3, generator=torch.Generator("cuda").manual_seed(1))
        ctx.view(v, 0).uniform_(1e-4, 1e-3, generator=torch.Generator("cuda").manual_seed(2))

    hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=_lib.LAMB_ONCHIP)
    out = {}
    reset()
    for hold in (None, 11, 7, 5):
        for nosync in (False, True):
            os.environ.pop("COCONET_LAMB_OC_HOLD", None)
            if hold:
                os.environ["COCONET_LAMB_OC_HOLD"] = str(hold)
            os.environ["COCONET_LAMB_OC_NOSYNC"] = "1" if nosync else "0"
            for _ in range(3):
                fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
            torch.cuda.synchronize()
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record()
            for _ in range(20):
                fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
            e.record()
            torch.cuda.synchronize()
            key = f"hold{hold or 'default'}{'_nosync' if nosync else ''}"
            out[key] = {"ms": s.elapsed_time(e) / 20, "spilled": tl.onchip_spilled()}
            print(key, out[key], flush=True)
    os.environ.pop("COCONET_LAMB_OC_HOLD", None)
    os.environ.pop("COCONET_LAMB_OC_NOSYNC", None)
    ctx.check()
    Path("gpurun_out").mkdir(exist_ok=True)
    Path("gpurun_out/lamb_hold_probe.json").write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
