import sys, torch, numpy as np
sys.path.insert(0, ".")
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import BdrHParams, mm_overlap_fused_ar, matmul
from paper_2105_05720_b200.runtime import Context
from oracle import coconet_oracle as co
W, rows, H = 1, 256, 512
dtype = torch.bfloat16
ctx = Context(W, heap_bytes=64 << 20, timeout_ms=3000)
k = H // W
x, w = ctx.alloc([rows, k], dtype), ctx.alloc([k, H], dtype)
part, bb, rr, out = ctx.alloc([rows, H], dtype), ctx.alloc([H], dtype), ctx.alloc([rows, H], dtype), ctx.alloc([rows, H], dtype)
for r in range(W):
    ctx.view(x, r).normal_(); ctx.view(w, r).normal_(); ctx.view(bb, r).zero_(); ctx.view(rr, r).zero_()
heap = ctx._heap(0)
PAD = 4 * 8 * 8 * 2048 * 4
GA = (8 << 20) // 4
flags_off = PAD + GA - (128 << 10)
cnt_off = PAD + GA - (64 << 10)
def dump(tag):
    torch.cuda.synchronize()
    fl = heap[flags_off:flags_off + 64].view(torch.int32).cpu().tolist()
    cn = heap[cnt_off:cnt_off + 16].view(torch.int32).cpu().tolist()
    print(tag, "flags", fl[:8], "cnt", cn[:2], flush=True)
dump("before")
hp = BdrHParams(0.1, 5, co.fnv1a("dropout"), _lib.MATH_FAST)
try:
    mm_overlap_fused_ar(ctx, x, w, bb, rr, part, out, hp)
    ctx.check()
    print("call ok")
except Exception as e:
    print("ERR", e)
dump("after")
torch.cuda.synchronize()
print("part sample", ctx.view(part, 0)[0, :4].float().tolist(), "ref", (ctx.view(x,0).float() @ ctx.view(w,0).float())[0,:4].tolist())
print("out sample", ctx.view(out, 0)[0, :4].float().tolist())
# variant: run on a non-default torch stream
s2 = torch.cuda.Stream()
with torch.cuda.stream(s2):
    try:
        mm_overlap_fused_ar(ctx, x, w, bb, rr, part, out, hp)
        ctx.check(s2)
        print("nondefault stream call ok")
    except Exception as e:
        print("nondefault ERR", e)
dump("after2")
