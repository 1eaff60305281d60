"""Runs the BERT-336M LAMB step a few times with one schedule (for ncu).
Usage: python tools/lamb_one.py SCHED CAP WAVE [STEPS]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import LambHParams, TensorList, fused_rs_lamb_ag  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from paper_2105_05720_b200.workloads import bert_large_counts  # noqa: E402

sched = {"grid": _lib.LAMB_GRID, "stream": _lib.LAMB_STREAMED, "tma": _lib.LAMB_TMA}[sys.argv[1]]
cap, wave = int(sys.argv[2]), int(sys.argv[3])
steps = int(sys.argv[4]) if len(sys.argv) > 4 else 4
counts = bert_large_counts()
N = sum(counts)
ctx = Context(1, heap_bytes=N * 30 + (1 << 30))
tl = TensorList(ctx, counts, bucket_cap=cap)
grads = [ctx.alloc([n], torch.float16) for n in counts]
params = [ctx.alloc([n]) for n in counts]
m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
for i in range(len(counts)):
    ctx.view(grads[i], 0).normal_()
    ctx.view(params[i], 0).uniform_(0.1, 0.9)
ctx.view(m, 0).zero_()
ctx.view(v, 0).fill_(1e-3)
hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, sched=sched, lag_elems=wave)
for _ in range(steps):
    fused_rs_lamb_ag(ctx, tl, grads, params, m, v, hp)
ctx.check()
print("ok")
