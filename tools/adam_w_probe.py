"""BERT-336M fused Adam (fp16 g, 16384-element buckets) at W virtual ranks
on one B200: the LDG kernel against the TMA ring (local m/v/p through bulk
copies; across ranks g pulled and p pushed by the consumers), FAST and EXACT.
Bytes per global element summed over ranks: g from W ranks (2W), m/v/p read
(12), m/v written (8), p into W copies (4W).
Usage: python tools/adam_w_probe.py [W ...]"""
import json
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import AdamHParams, TensorList, fused_rs_adam_ag  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from paper_2105_05720_b200.workloads import bert_large_counts  # noqa: E402
from tools.pattern_probe import timeit  # noqa: E402

counts = bert_large_counts()
N = sum(counts)
for W in [int(x) for x in sys.argv[1:]] or [1, 2, 4, 8]:
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
    row = {}
    for math, mn in ((_lib.MATH_FAST, "fast"), (_lib.MATH_EXACT, "exact")):
        hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, math, _lib.ALGO_TWO_SHOT)
        for impl, env, ctas in (("ldg", "0", "3"), ("tma", "1", "3"), ("tma_ring3", "1", "2")):
            os.environ["COCONET_ADAM_TMA"] = env
            os.environ["COCONET_ADAM_TMA_CTAS"] = ctas
            ms = timeit(lambda: fused_rs_adam_ag(ctx, tl, grads, params, m, v, hp), 5, warmup=2)
            row[f"{mn}_{impl}_ms"] = round(ms, 3)
            row[f"{mn}_{impl}_GBs"] = round((20 + 6 * W) * N / ms / 1e6, 1)
    os.environ.pop("COCONET_ADAM_TMA", None)
    os.environ.pop("COCONET_ADAM_TMA_CTAS", None)
    print(json.dumps({f"W{W}": row}), flush=True)
    ctx.close()
