"""One-shot vs two-shot fused Adam (and tensor-list AllReduce) by message
size on one B200 with virtual ranks: the data behind AUTO's crossover
(paper: 2^16 on V100). Usage: python tools/crossover_probe.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import AdamHParams, TensorList, allreduce, fused_rs_adam_ag  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from tools.pattern_probe import timeit  # noqa: E402

out = {}
for W in (2, 4, 8):
    for lg in range(12, 23, 2):
        N = 1 << lg
        ctx = Context(W, heap_bytes=N * 40 + (64 << 20))
        tl = TensorList(ctx, [N])
        g, p = ctx.alloc([N]), ctx.alloc([N])
        st = max(tl.state_elems, tl.shard_elems)
        m, v = ctx.alloc([st]), ctx.alloc([st])
        o = ctx.alloc([N])
        for r in range(W):
            ctx.view(g, r).normal_()
            ctx.view(p, r).uniform_(0.1, 0.9)
            ctx.view(m, r).zero_()
            ctx.view(v, r).fill_(1e-3)
        row = {}
        for algo, an in ((_lib.ALGO_ONE_SHOT, "one"), (_lib.ALGO_TWO_SHOT, "two")):
            hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, _lib.MATH_FAST, algo)
            row[f"adam_{an}_us"] = round(timeit(lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp), 30) * 1e3, 2)
            row[f"ar_{an}_us"] = round(timeit(lambda: allreduce(ctx, tl, [g], [o], algo=algo), 30) * 1e3, 2)
        out[f"W{W}_N2^{lg}"] = row
        print(json.dumps({f"W{W}_N2^{lg}": row}), flush=True)
        ctx.close()
