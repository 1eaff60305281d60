"""LAMB schedule probe (not the bench): GRID vs STREAMED (several L2 wave
sizes, bucket capacities) on the BERT-336M list at W=1, fp16 grads; CUDA-event
times and bit-identity of one step against GRID.
Usage: python tools/lamb_probe.py [--steps K]"""
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
    ap.add_argument("--caps", default="1024,4096")
    ap.add_argument("--waves", default="")
    args = ap.parse_args()
    counts = bert_large_counts()
    N = sum(counts)
    out = {"N": N}
    ctx = Context(1, heap_bytes=N * 30 + (1 << 30))
    for cap in [int(c) for c in args.caps.split(",")]:
        tl = TensorList(ctx, counts, bucket_cap=cap)
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
            return torch.cat([ctx.view(p, 0) for p in params] + [ctx.view(m, 0), ctx.view(v, 0)]).clone()

        ref = None
        configs = [("grid", _lib.LAMB_GRID, 0), ("tma", _lib.LAMB_TMA, 0)] + [
            (f"stream_lag{w}", _lib.LAMB_STREAMED, int(w)) for w in args.waves.split(",") if w]
        for name, sched, wave in configs:
            hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched, lag_elems=wave)
            reset()
            fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
            ctx.check()
            snap = snapshot()
            if ref is None:
                ref = snap
            same = bool(torch.equal(snap, ref))
            snap_f = snap
            ms = timeit(lambda: fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp), args.steps)
            ctx.check()
            out[f"cap{cap}_{name}"] = {"ms": ms, "GBs_at_26B": 26 * N / ms / 1e6,
                                       "GBs_at_38B": 38 * N / ms / 1e6, "bit_identical_to_grid": same,
                                       "max_abs_diff_vs_grid": float((snap_f - ref).abs().max()),
                                       "lag": wave if sched == _lib.LAMB_STREAMED else None}
            print(json.dumps({f"cap{cap}_{name}": out[f"cap{cap}_{name}"]}), flush=True)
        del ref
        tl.close()
        ctx.reset()
    ctx.close()
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
