"""ONCHIP LAMB probe (not the bench): the TMA schedule vs ONCHIP at several
head depths / ring sizes on the BERT-336M list at W=1, fp16 grads, 16384-
element buckets; CUDA-event times, and one step's p, m, v against TMA.
Usage: python tools/lamb_oc_probe.py [--heads 4,6,8] [--stages 3,4]"""
import argparse
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
from tools.probe import timeit  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--cap", type=int, default=16384)
    ap.add_argument("--heads", default="6")
    ap.add_argument("--stages", default="4")
    ap.add_argument("--slots", default="")
    ap.add_argument("--shapes", default="162", help="consumer warps x quads per thread: 162, 161, 82")
    ap.add_argument("--head2s", default="")
    ap.add_argument("--out", default="")
    args = ap.parse_args()
    counts = bert_large_counts()
    N = sum(counts)
    out = {"N": N, "cap": args.cap}
    ctx = Context(1, heap_bytes=N * 16 + (1 << 30))
    tl = TensorList(ctx, counts, bucket_cap=args.cap)
    grads = [ctx.alloc([n], torch.float16) for n in counts]
    params = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])

    def reset():
        for i, n in enumerate(counts):
            gen_values(ctx, ctx.view(grads[i], 0), 1, f"g{i}", "local", 0, [n], group_size=1)
            gen_values(ctx, ctx.view(params[i], 0), 1, f"p{i}", "replicated", 0, [n], group_size=1)
        ctx.view(m, 0).uniform_(-1e-3, 1e-3, generator=torch.Generator("cuda").manual_seed(1))
        ctx.view(v, 0).uniform_(1e-4, 1e-3, generator=torch.Generator("cuda").manual_seed(2))

    def snapshot():
        return (torch.cat([ctx.view(p, 0) for p in params]).clone(), ctx.view(m, 0).clone(), ctx.view(v, 0).clone())

    ref = None
    configs = [("tma", _lib.LAMB_TMA, None, None, None)]
    for w in args.shapes.split(","):
        for h in args.heads.split(","):
            for s in args.stages.split(","):
                for x in (args.slots.split(",") if args.slots else [None]):
                    for h2 in (args.head2s.split(",") if args.head2s else [None]):
                        configs.append((f"onchip_shape{w}_head{h}_stages{s}" + (f"_slots{x}" if x else "")
                                        + (f"_head2_{h2}" if h2 else ""), _lib.LAMB_ONCHIP, h, s, x, w, h2))
    for name, sched, head, stages, slots, *wr in configs:
        for k, val in (("COCONET_LAMB_OC_HEAD", head), ("COCONET_LAMB_OC_STAGES", stages),
                       ("COCONET_LAMB_OC_SMEM_SLOTS", slots), ("COCONET_LAMB_OC_SHAPE", wr[0] if wr else None),
                       ("COCONET_LAMB_OC_HEAD2", wr[1] if len(wr) > 1 else None)):
            if val is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = val
        hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched)
        reset()
        fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
        ctx.check()
        snap = snapshot()
        if ref is None:
            ref = snap
        p_dev = float(((snap[0] - ref[0]).abs().max() / ref[0].abs().max()).item())
        mv_same = bool(torch.equal(snap[1], ref[1]) and torch.equal(snap[2], ref[2]))
        ms = timeit(lambda: fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp), args.steps)
        ctx.check()
        out[name] = {"ms": ms, "GBs_at_38B": 38 * N / ms / 1e6, "GBs_at_26B": 26 * N / ms / 1e6,
                     "p_rel_dev_vs_tma": p_dev, "m_v_bit_identical_to_tma": mv_same}
        print(json.dumps({name: out[name]}), flush=True)
    ctx.close()
    print(json.dumps(out, indent=1))
    if args.out:
        Path(args.out).write_text(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
