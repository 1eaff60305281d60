"""Where the small-message floor of the fused Adam / AllReduce calls goes:
host call rate (back-to-back calls, CUDA events) against the kernel's own
device duration (torch.profiler / CUPTI). Usage: python tools/floor_probe.py"""
import json
import sys
import time
from pathlib import Path

import torch
from torch.profiler import ProfilerActivity, profile

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import AdamHParams, TensorList, allreduce, fused_rs_adam_ag  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from tools.pattern_probe import timeit  # noqa: E402


def device_us(fn, n=30):
    fn()
    torch.cuda.synchronize()
    with profile(activities=[ProfilerActivity.CUDA]) as prof:
        for _ in range(n):
            fn()
        torch.cuda.synchronize()
    ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
    tot = {}
    for e in ev:
        tot.setdefault(e.name, []).append(e.device_time)
    return {k[:60]: round(sum(v) / len(v), 2) for k, v in tot.items()}


def host_us(fn, n=200):
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        fn()
    h = (time.perf_counter() - t) / n * 1e6
    torch.cuda.synchronize()
    return round(h, 2)


for W, lg in ((1, 12), (4, 12), (4, 20), (8, 16)):
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
    hp = AdamHParams(1e-3, 0.9, 0.999, 1.0, 1e-8, False, _lib.MATH_FAST, _lib.ALGO_TWO_SHOT)
    fa = lambda: fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp)  # noqa: E731
    fr = lambda: allreduce(ctx, tl, [g], [o], algo=_lib.ALGO_TWO_SHOT)  # noqa: E731
    from paper_2105_05720_b200.collectives import _ptrs
    import ctypes as C
    args = (ctx.handle, tl.handle, _ptrs(ctx, [g]), _lib.F32, _ptrs(ctx, [p]),
            ctx.ptr(m), ctx.ptr(v), C.byref(_lib.AdamParams(hp.lr, hp.beta1, hp.beta2, hp.t, hp.eps, 0, hp.math,
                                                            hp.algo)), ctx.stream_ptr(None))
    fraw = lambda: ctx.lib.coconet_fused_rs_adam_ag(*args)  # noqa: E731
    row = {"adam_raw_host_us": host_us(fraw), "adam_raw_event_us": round(timeit(fraw, 30) * 1e3, 2),
           "adam_event_us": round(timeit(fa, 30) * 1e3, 2), "adam_host_us": host_us(fa),
           "adam_kernels": device_us(fa),
           "ar_event_us": round(timeit(fr, 30) * 1e3, 2), "ar_host_us": host_us(fr), "ar_kernels": device_us(fr)}
    print(json.dumps({f"W{W}_N2^{lg}": row}), flush=True)
    ctx.close()
