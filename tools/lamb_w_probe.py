"""BERT-336M fused LAMB at W = 2/4/8 VIRTUAL ranks on one B200: GRID (LDG)
against TMA (local m/v/p through the bulk-copy ring, g pulled and p pushed
across ranks by the consumers). Bytes summed over ranks per global element:
g from W ranks (2W), m/v/p + m/v (20), m/v/p (12), p into W copies (4W).
Usage: python tools/lamb_w_probe.py [W ...]   (COCONET_PROBE_CAP: bucket cap, default 16384)"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import LambHParams, TensorList, fused_rs_lamb_ag  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from paper_2105_05720_b200.workloads import bert_large_counts  # noqa: E402
from tools.pattern_probe import timeit  # noqa: E402

counts = bert_large_counts()
N = sum(counts)
for W in [int(x) for x in sys.argv[1:]] or [2, 4, 8]:
    ctx = Context(W, heap_bytes=N * 6 + 2 * (N // W + 64 * len(counts) + 4096) * 4 + (512 << 20))
    tl = TensorList(ctx, counts, bucket_cap=int(os.environ.get("COCONET_PROBE_CAP", 16384)))
    grads = [ctx.alloc([n], torch.float16) for n in counts]
    params = [ctx.alloc([n]) for n in counts]
    m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
    for r in range(W):
        for i, n in enumerate(counts):
            ctx.view(grads[i], r).normal_()
            ctx.view(params[i], r).uniform_(0.1, 0.9)
        ctx.view(m, r).zero_()
        ctx.view(v, r).fill_(1e-3)
    row = {}
    # COCONET_LAMB_TMA_CTAS sizes the ring as for that many CTAs per SM
    # (2 stay resident at W > 1: registers): 1 -> 7 stages, 2 -> 3, 3 -> 2
    for name, sched, ctas in (("grid", _lib.LAMB_GRID, None), ("tma", _lib.LAMB_TMA, None),
                              ("tma_1cta", _lib.LAMB_TMA, "1"), ("tma_ring2", _lib.LAMB_TMA, "3")):
        if ctas:
            os.environ["COCONET_LAMB_TMA_CTAS"] = ctas
        hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched)
        ms = timeit(lambda: fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp), 5, warmup=2)
        os.environ.pop("COCONET_LAMB_TMA_CTAS", None)
        row[f"{name}_ms"] = round(ms, 3)
        row[f"{name}_GBs"] = round((32 + 6 * W) * N / ms / 1e6, 1)
    print(json.dumps({f"W{W}": row}), flush=True)
    ctx.close()
