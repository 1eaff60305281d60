"""Python wrappers of the fused compute/communication entry points.

Every function is collective over its group and asynchronous on the current
torch stream; buffers are `SymmBuffer`s of the context (same offset on every
rank). See include/coconet_cuda.h for the reference routine each one replaces.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from ._lib import check, i64_array, ptr_array
from .runtime import Context, SymmBuffer, elem_of

FNV_OFFSET = 0xcbf29ce484222325
FNV_PRIME = 0x100000001b3


def fnv1a(s: str | bytes, h: int = FNV_OFFSET) -> int:
    """ccopt::fnv1a (types.hpp:161-170) — decl keys, dropout keys."""
    data = s.encode() if isinstance(s, str) else s
    for b in data:
        h ^= b
        h = (h * FNV_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


class TensorList:
    """Device bucket table (BucketTable, runtime.hpp:575-614) for a list of
    tensors with element counts `counts`, on group `group`."""

    def __init__(self, ctx: Context | None, counts, group: int = 0, bucket_cap: int = 1024,
                 world: int | None = None):
        """ctx=None builds a host-only plan for `world` ranks (no device)."""
        self.ctx = ctx
        self.counts = [int(c) for c in counts]
        self.group = group
        h = C.c_void_p()
        lib = ctx.lib if ctx is not None else _lib.load()
        self.lib = lib
        if ctx is None:
            check(lib.coconet_tlist_plan(int(world), len(self.counts), i64_array(self.counts),
                                         bucket_cap, C.byref(h)))
        else:
            check(lib.coconet_tlist_create(ctx.handle, group, len(self.counts),
                                           i64_array(self.counts), bucket_cap, C.byref(h)))
        self.handle = h
        self.total = int(lib.coconet_tlist_total(h))
        self.shard_elems = int(lib.coconet_tlist_shard_elems(h))
        self.state_elems = int(lib.coconet_tlist_state_elems(h))
        self.n_buckets = int(lib.coconet_tlist_buckets(h))
        self.metadata_bytes = int(lib.coconet_tlist_metadata_bytes(h))

    def chunk(self, r: int) -> tuple[int, int]:
        lo, hi = C.c_int64(), C.c_int64()
        check(self.lib.coconet_tlist_chunk(self.handle, r, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def segments(self, r: int) -> np.ndarray:
        """[n, 4] int64 (tensor, toff, len, state index) of rank r's segments
        (r = -1: the ONE_SHOT table)."""
        n = self.n_buckets + 16
        bufs = [(C.c_int64 * n)() for _ in range(4)]
        got = int(self.lib.coconet_tlist_segments(self.handle, r, *bufs, n))
        check(0 if got >= 0 else 3)
        return np.stack([np.frombuffer(b, dtype=np.int64)[:got] for b in bufs], axis=1)

    def stream_items(self, lag: int, r: int) -> np.ndarray:
        """[n, 4] int64 (tensor, toff, len, pass) of rank r's STREAMED-LAMB work
        list for a pass-1 -> pass-2 lag of `lag` elements, in execution order."""
        n = 2 * (self.n_buckets + 16 * _lib.MAX_RANKS)
        bufs = [(C.c_int64 * n)() for _ in range(4)]
        got = int(self.lib.coconet_tlist_stream_items(self.handle, int(lag), r, *bufs, n))
        check(0 if got >= 0 else 3)
        return np.stack([np.frombuffer(b, dtype=np.int64)[:got] for b in bufs], axis=1)

    def onchip_spilled(self) -> int:
        """Elements the last ONCHIP-LAMB launch did not hold on chip (past the hold or cover items; -1: no plan)."""
        return int(self.lib.coconet_tlist_onchip_spilled(self.handle))

    def state_index_map(self, r: int):
        """(tensor, element, state index) arrays of every element rank r owns."""
        segs = self.segments(r)
        if len(segs) == 0:
            z = np.zeros(0, np.int64)
            return z, z, z
        lens = segs[:, 2]
        rep = np.repeat(np.arange(len(segs)), lens)
        within = np.arange(int(lens.sum())) - np.repeat(np.cumsum(lens) - lens, lens)
        return segs[rep, 0], segs[rep, 1] + within, segs[rep, 3] + within

    def shard_index(self, pos: int) -> int:
        return int(self.lib.coconet_tlist_shard_index(self.handle, pos))

    def close(self):
        if self.handle:
            self.lib.coconet_tlist_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _ptrs(ctx: Context, bufs):
    """The C pointer array of `bufs` (rank 0's heap in VIRTUAL mode), built
    once per buffer list: a training loop passes the same list every step."""
    key = tuple(b.offset for b in bufs)
    cache = ctx.__dict__.setdefault("_ptr_arrays", {})
    arr = cache.get(key)
    if arr is None:
        if len(cache) > 256:
            cache.clear()
        arr = cache[key] = ptr_array([ctx.ptr(b) for b in bufs])
    return arr


@dataclass
class AdamHParams:
    lr: float
    beta1: float
    beta2: float
    t: float
    eps: float = 0.0
    cv_beta1: bool = True   # the golden's (1-beta1) second-moment coefficient
    math: int = _lib.MATH_EXACT
    algo: int = _lib.ALGO_AUTO


@dataclass
class LambHParams:
    lr: float
    beta1: float
    beta2: float
    t: float
    eps: float = 1e-6
    wd: float = 0.01
    math: int = _lib.MATH_FAST
    sched: int = _lib.LAMB_AUTO   # GRID or STREAMED (L2-resident pass 2); results are bit-identical
    lag_elems: int = 0            # STREAMED: pass-1 -> pass-2 distance in elements (0 = library default)
    trust_guard: bool = False     # ratio = lr for a zero-norm tensor (apex/NVLAMB); False = the golden's formula


def fused_rs_adam_ag(ctx: Context, tl: TensorList, grads, params, m: SymmBuffer, v: SymmBuffer,
                     hp: AdamHParams, stream=None) -> None:
    """ReduceScatter + Adam + AllGather (FusedAllReduce, runtime.hpp:471-516)."""
    g_elem = elem_of(grads[0].dtype)
    p = _lib.AdamParams(hp.lr, hp.beta1, hp.beta2, hp.t, hp.eps, int(hp.cv_beta1), hp.math, hp.algo)
    check(ctx.lib.coconet_fused_rs_adam_ag(
        ctx.handle, tl.handle, _ptrs(ctx, grads), g_elem, _ptrs(ctx, params), ctx.ptr(m), ctx.ptr(v),
        C.byref(p), ctx.stream_ptr(stream)))


def fused_rs_lamb_ag(ctx: Context, tl: TensorList, grads, params, m: SymmBuffer, v: SymmBuffer,
                     hp: LambHParams, stream=None) -> None:
    g_elem = elem_of(grads[0].dtype)
    p = _lib.LambParams(hp.lr, hp.beta1, hp.beta2, hp.t, hp.eps, hp.wd, hp.math, hp.sched, hp.lag_elems,
                         int(hp.trust_guard))
    check(ctx.lib.coconet_fused_rs_lamb_ag(
        ctx.handle, tl.handle, _ptrs(ctx, grads), g_elem, _ptrs(ctx, params), ctx.ptr(m), ctx.ptr(v),
        C.byref(p), ctx.stream_ptr(stream)))


def unfused_lamb(ctx: Context, tl: TensorList, grads, params, m: SymmBuffer, v: SymmBuffer, u: SymmBuffer,
                 norms: torch.Tensor, hp: LambHParams, stream=None) -> None:
    """The "separate kernels" baseline (coconet_unfused_lamb): apex FusedLAMB's
    four multi-tensor passes over a size-1 group's list. `norms` is a device
    float64 tensor of 2 * n_tensors."""
    g_elem = elem_of(grads[0].dtype)
    p = _lib.LambParams(hp.lr, hp.beta1, hp.beta2, hp.t, hp.eps, hp.wd, hp.math, hp.sched, hp.lag_elems,
                        int(hp.trust_guard))
    check(ctx.lib.coconet_unfused_lamb(
        ctx.handle, tl.handle, _ptrs(ctx, grads), g_elem, _ptrs(ctx, params), ctx.ptr(m), ctx.ptr(v), ctx.ptr(u),
        C.c_void_p(norms.data_ptr()), C.byref(p), ctx.stream_ptr(stream)))


def send(ctx: Context, src_group: int, dst_group: int, x: SymmBuffer, out: SymmBuffer, stream=None) -> None:
    """Send/Recv (runtime.hpp:439-470): group rank r of src_group stores its x
    into out on group rank r of dst_group."""
    check(ctx.lib.coconet_send(ctx.handle, src_group, dst_group, ctx.ptr(x), ctx.ptr(out), elem_of(x.dtype),
                               x.numel, ctx.stream_ptr(stream)))


def allreduce(ctx: Context, tl: TensorList, xs, outs, reducer: int = _lib.SUM,
              algo: int = _lib.ALGO_AUTO, stream=None) -> None:
    """Tensor-list AllReduce (runtime.hpp:384-395; scattered_collective :624-675)."""
    check(ctx.lib.coconet_allreduce(ctx.handle, tl.handle, _ptrs(ctx, xs), _ptrs(ctx, outs),
                                    elem_of(xs[0].dtype), reducer, algo, ctx.stream_ptr(stream)))


def reduce_scatter(ctx: Context, x: SymmBuffer, out: SymmBuffer, axis: int = -1, group: int = 0,
                   reducer: int = _lib.SUM, stream=None) -> None:
    shape = i64_array(x.shape)
    check(ctx.lib.coconet_reduce_scatter(ctx.handle, group, ctx.ptr(x), ctx.ptr(out),
                                         elem_of(x.dtype), reducer, len(x.shape), shape,
                                         axis if axis >= 0 else len(x.shape) - 1,
                                         ctx.stream_ptr(stream)))


def all_gather(ctx: Context, x: SymmBuffer | None, out: SymmBuffer, axis: int = -1, group: int = 0,
               stream=None) -> None:
    shape = i64_array(out.shape)
    check(ctx.lib.coconet_all_gather(ctx.handle, group, ctx.ptr(x) if x is not None else None,
                                     ctx.ptr(out), elem_of(out.dtype), len(out.shape), shape,
                                     axis if axis >= 0 else len(out.shape) - 1,
                                     ctx.stream_ptr(stream)))


def reduce(ctx: Context, x: SymmBuffer, out: SymmBuffer, root: int = 0, reducer: int = _lib.SUM,
           group: int = 0, stream=None) -> None:
    """Reduce to `root` (runtime.hpp:415-428): rank-order fp32 fold on the
    root, zeros elsewhere."""
    check(ctx.lib.coconet_reduce(ctx.handle, group, ctx.ptr(x), ctx.ptr(out), elem_of(x.dtype), reducer,
                                 x.numel, root, ctx.stream_ptr(stream)))


def broadcast(ctx: Context, x: SymmBuffer, out: SymmBuffer, root: int = 0, group: int = 0, stream=None) -> None:
    """Broadcast from `root` (runtime.hpp:429-436)."""
    check(ctx.lib.coconet_broadcast(ctx.handle, group, ctx.ptr(x), ctx.ptr(out), elem_of(x.dtype), x.numel, root,
                                    ctx.stream_ptr(stream)))


def gen_values(ctx: Context, dst: torch.Tensor, seed: int, name: str, layout: str, rank: int,
               global_shape, sliced_dim: int = -1, group_size: int = 1, stream=None) -> None:
    """gen_decl_values (state.hpp:55-74) for one decl on one rank, on device."""
    shape = i64_array(global_shape)
    check(ctx.lib.coconet_gen_values(ctx.handle, C.c_void_p(dst.data_ptr()), elem_of(dst.dtype),
                                     seed & 0xFFFFFFFFFFFFFFFF, fnv1a(name), int(layout == "local"),
                                     rank, len(global_shape), shape, sliced_dim, group_size,
                                     ctx.stream_ptr(stream)))


@dataclass
class BdrHParams:
    rate: float
    seed: int
    key: int
    math: int = _lib.MATH_EXACT

    def c(self):
        return _lib.BdrParams(self.rate, self.seed, self.key, self.math)


def fused_rs_bdr_ag(ctx: Context, x: SymmBuffer, b: SymmBuffer, r: SymmBuffer, out: SymmBuffer,
                    hp: BdrHParams, group: int = 0, stream=None) -> None:
    rows = int(np.prod(x.shape[:-1])) if len(x.shape) > 1 else 1
    p = hp.c()
    check(ctx.lib.coconet_fused_rs_bdr_ag(ctx.handle, group, ctx.ptr(x), ctx.ptr(b), ctx.ptr(r),
                                          ctx.ptr(out), elem_of(x.dtype), rows, x.shape[-1],
                                          C.byref(p), ctx.stream_ptr(stream)))


def rs_fused_send_ag(ctx: Context, src_group: int, dst_group: int, x: SymmBuffer, b: SymmBuffer,
                     r: SymmBuffer, out: SymmBuffer, hp: BdrHParams, stream=None) -> None:
    p = hp.c()
    check(ctx.lib.coconet_rs_fused_send_ag(ctx.handle, src_group, dst_group, ctx.ptr(x), ctx.ptr(b),
                                           ctx.ptr(r), ctx.ptr(out), elem_of(x.dtype), x.numel,
                                           C.byref(p), ctx.stream_ptr(stream)))


def matmul(ctx: Context, a: SymmBuffer, b: SymmBuffer, c: SymmBuffer, math: int = _lib.MATH_FAST,
           group: int = 0, stream=None) -> None:
    m = int(np.prod(a.shape[:-1]))
    k = a.shape[-1]
    n = b.shape[-1]
    check(ctx.lib.coconet_matmul(ctx.handle, group, ctx.ptr(a), ctx.ptr(b), ctx.ptr(c),
                                 elem_of(a.dtype), elem_of(c.dtype), m, n, k, math,
                                 ctx.stream_ptr(stream)))


def mm_overlap_fused_ar(ctx: Context, a: SymmBuffer, w: SymmBuffer, b: SymmBuffer, r: SymmBuffer,
                        partial: SymmBuffer, out: SymmBuffer, hp: BdrHParams, group: int = 0,
                        stream=None) -> None:
    rows = int(np.prod(a.shape[:-1]))
    p = hp.c()
    check(ctx.lib.coconet_mm_overlap_fused_ar(ctx.handle, group, ctx.ptr(a), ctx.ptr(w), ctx.ptr(b),
                                              ctx.ptr(r), ctx.ptr(partial), ctx.ptr(out),
                                              elem_of(a.dtype), rows, w.shape[-1], a.shape[-1],
                                              C.byref(p), ctx.stream_ptr(stream)))


class LambHostPipeline:
    """A fused RS+LAMB+AG step whose gradients come from, and whose updated
    parameters go back to, pinned HOST memory (the reference's own contract:
    Engine::run takes and returns host vectors, runtime.hpp:101).

    LAMB's trust ratio is per tensor, so the tensor list is cut into `groups`
    contiguous tensor groups of about equal size, each with its own bucket
    table and state shard. Per step, group k's H2D copy (one contiguous
    range of the flat gradient buffer), its fused launch and its D2H copy run
    on three streams, so PCIe in both directions overlaps the kernels:
        H2D(k+1) || LAMB(k) || D2H(k-1).
    Results are those of one fused step over the whole list (W = 1: bitwise;
    W > 1: every element reduced in its own group's ring order).

    counts: element counts; g_flat / p_flat: symmetric flat buffers holding the
    tensors at `offsets` (elements, 4-aligned); host buffers passed to step()
    use the same flat layout."""

    def __init__(self, ctx: Context, counts, g_flat: SymmBuffer, p_flat: SymmBuffer, offsets, groups: int = 8,
                 bucket_cap: int = 4096):
        self.ctx = ctx
        counts = [int(c) for c in counts]
        offsets = [int(o) for o in offsets]
        total = sum(counts)
        gsz = torch.empty((), dtype=g_flat.dtype).element_size()
        cuts, acc = [0], 0
        for i, n in enumerate(counts):
            acc += n
            if acc * groups >= total * len(cuts) and i + 1 < len(counts) and len(cuts) < groups:
                cuts.append(i + 1)
        cuts.append(len(counts))
        self.groups = []
        for a, b in zip(cuts[:-1], cuts[1:]):
            if a == b:
                continue
            tl = TensorList(ctx, counts[a:b], bucket_cap=bucket_cap)
            grads = [SymmBuffer(g_flat.offset + offsets[i] * gsz, (counts[i],), g_flat.dtype) for i in range(a, b)]
            params = [SymmBuffer(p_flat.offset + offsets[i] * 4, (counts[i],), torch.float32) for i in range(a, b)]
            lo, hi = offsets[a], offsets[b - 1] + counts[b - 1]
            m = ctx.alloc([tl.shard_elems], torch.float32)
            v = ctx.alloc([tl.shard_elems], torch.float32)
            self.groups.append(dict(tl=tl, grads=grads, params=params, lo=lo, hi=hi, m=m, v=v))
        # launch order: the smallest group first (the D2H stream starts
        # early) and the next smallest last (the final D2H, which nothing
        # overlaps, is short); the rest in list order
        if len(self.groups) > 2 and os.environ.get("COCONET_E2E_ORDER", "small_ends") == "small_ends":
            by_size = sorted(range(len(self.groups)), key=lambda i: self.groups[i]["hi"] - self.groups[i]["lo"])
            first, last = by_size[0], by_size[1]
            mid = [i for i in range(len(self.groups)) if i not in (first, last)]
            self.groups = [self.groups[i] for i in [first] + mid + [last]]
        self.g_flat, self.p_flat = g_flat, p_flat
        self.h2d = torch.cuda.Stream(device=ctx.device)
        self.d2h = torch.cuda.Stream(device=ctx.device)
        self.ev_in = [torch.cuda.Event() for _ in self.groups]
        self.ev_run = [torch.cuda.Event() for _ in self.groups]
        self.ev_out = [torch.cuda.Event() for _ in self.groups]
        self.stepped = False
        self.h2d_bytes = sum(g["hi"] - g["lo"] for g in self.groups) * gsz
        self.d2h_bytes = sum(g["hi"] - g["lo"] for g in self.groups) * 4

    def state(self):
        """(m, v) shard buffers of every group (for initialisation)."""
        return [(g["m"], g["v"]) for g in self.groups]

    def step(self, h_grads: torch.Tensor, h_params: torch.Tensor, hp: LambHParams, stream=None) -> None:
        """h_grads / h_params: pinned flat host tensors (the flat layout of
        g_flat / p_flat). Asynchronous; h_params is complete once
        `self.d2h` is (see wait())."""
        ctx = self.ctx
        comp = stream if stream is not None else torch.cuda.current_stream()
        dg = ctx.view(self.g_flat)
        dp = ctx.view(self.p_flat)
        for k, g in enumerate(self.groups):
            with torch.cuda.stream(self.h2d):
                if self.stepped:  # the previous step's launch must be done reading these gradients
                    self.h2d.wait_event(self.ev_run[k])
                dg[g["lo"]:g["hi"]].copy_(h_grads[g["lo"]:g["hi"]], non_blocking=True)
                self.ev_in[k].record(self.h2d)
            comp.wait_event(self.ev_in[k])
            if self.stepped:  # the previous step's D2H of these params must be done before we overwrite them
                comp.wait_event(self.ev_out[k])
            fused_rs_lamb_ag(ctx, g["tl"], g["grads"], g["params"], g["m"], g["v"], hp, stream=comp)
            self.ev_run[k].record(comp)
            with torch.cuda.stream(self.d2h):
                self.d2h.wait_event(self.ev_run[k])
                h_params[g["lo"]:g["hi"]].copy_(dp[g["lo"]:g["hi"]], non_blocking=True)
                self.ev_out[k].record(self.d2h)
        self.stepped = True

    def wait(self):
        self.d2h.synchronize()
