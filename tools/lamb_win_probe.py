"""WINDOWED LAMB probe (not the bench): the TMA schedule vs the WINDOWED one
at several window sizes on the BERT-336M list at W=1, fp16 grads, 16384-
element buckets; CUDA-event times, and one step's p, m, v against TMA.
Usage: python tools/lamb_win_probe.py [--wins 1048576,2097152,...]"""
import argparse
import json
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
    ap.add_argument("--wins", default="1048576,2097152,4194304,8388608,16777216")
    ap.add_argument("--heads", default="2")
    ap.add_argument("--hints", default="0")
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
    import os
    configs = [("tma", _lib.LAMB_TMA, 0, "2", "0")] + [
        (f"win{w}_head{h}_hints{x}", _lib.LAMB_WINDOWED, int(w), h, x)
        for w in args.wins.split(",") if w for h in args.heads.split(",") for x in args.hints.split(",")]
    for name, sched, win, head, hints in configs:
        os.environ["COCONET_LAMB_WIN_HEAD"] = head
        os.environ["COCONET_LAMB_WIN_HINTS"] = hints
        hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched, lag_elems=win)
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


if __name__ == "__main__":
    main()
