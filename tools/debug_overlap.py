import sys, torch
sys.path.insert(0, ".")
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import BdrHParams, mm_overlap_fused_ar
from paper_2105_05720_b200.runtime import Context
from oracle import coconet_oracle as co
W, rows, H = int(sys.argv[1]) if len(sys.argv) > 1 else 1, 256, 512
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
    cn = heap[cnt_off:cnt_off + 128].view(torch.int32).cpu().tolist()
    print(tag, "flags", fl[:8], "cnt", cn[0], "ticket", cn[16], flush=True)
dump("before")
hp = BdrHParams(0.1, 5, co.fnv1a("dropout"), _lib.MATH_FAST)
try:
    mm_overlap_fused_ar(ctx, x, w, bb, rr, part, out, hp)
    ctx.check()
    print("call ok")
except Exception as e:
    print("ERR", e)
dump("after")
print("part", ctx.view(part, 0)[0, :4].float().tolist(), "ref", (ctx.view(x,0).float() @ ctx.view(w,0).float())[0,:4].tolist())
print("out", ctx.view(out, 0)[0, :4].float().tolist())
