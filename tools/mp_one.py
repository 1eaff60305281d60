"""C3 model-parallel pattern on one GPU (8 virtual ranks) for ncu: runs the
plain GEMM, the fused RS-BDR-AG and the overlapped kernel `steps` times each.
Usage: python tools/mp_one.py [which=all|gemm|ar|overlap] [steps]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import BdrHParams, fused_rs_bdr_ag, matmul, mm_overlap_fused_ar  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "all"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
W, rows, H = 8, 8192, 3072
k = H // W
dt = torch.bfloat16
ctx = Context(W, heap_bytes=(3 << 30))
x, w = ctx.alloc([rows, k], dt), ctx.alloc([k, H], dt)
part, bb, rr, o1 = ctx.alloc([rows, H], dt), ctx.alloc([H], dt), ctx.alloc([rows, H], dt), ctx.alloc([rows, H], dt)
for r in range(W):
    ctx.view(x, r).normal_()
    ctx.view(w, r).normal_(0, k ** -0.5)
    ctx.view(bb, r).normal_(0, 0.1)
    ctx.view(rr, r).normal_()
hp = BdrHParams(0.1, 1, 11617925594314093840, _lib.MATH_FAST)
for _ in range(steps):
    if which in ("all", "gemm"):
        matmul(ctx, x, w, part, math=_lib.MATH_FAST)
    if which in ("all", "ar"):
        fused_rs_bdr_ag(ctx, part, bb, rr, o1, hp)
    if which in ("all", "overlap"):
        mm_overlap_fused_ar(ctx, x, w, bb, rr, part, o1, hp)
ctx.check()
print("ok")
