"""torch.optim integration of the fused data-parallel step (SURVEY §8(f)-2,
paper §5 "PyTorch integration").

`FusedAdam` / `FusedLAMB` re-home every parameter (and its .grad) into the
context's symmetric heap and build the bucket table once. `step()` is then one
fused ReduceScatter + optimizer + AllGather launch over the whole list:
- gradients are SUMMED across ranks, as the reference's AllReduce does
  (scale the loss by 1/world for a mean);
- optimizer state is sharded (ZeRO-1 style, the as_slice of m and v);
- updated parameters land in every rank's copy in place.

DISTRIBUTED mode: one process per GPU, `Context(world, "distributed", rank)`.
VIRTUAL mode with world 1 is a plain single-GPU fused optimizer.
"""
from __future__ import annotations

import torch

from . import _lib
from .collectives import AdamHParams, LambHParams, TensorList, fused_rs_adam_ag, fused_rs_lamb_ag
from .runtime import Context


def _rehome(ctx: Context, params, grad_dtype):
    """Moves each parameter's storage into the heap. With fp32 grads the .grad
    is a heap view too (backward writes what the kernel pulls); autograd only
    produces grads of the parameter's dtype, so for a 16-bit grad_dtype .grad
    stays an ordinary fp32 tensor and `_stage_grads` casts it into the 16-bit
    heap buffer before each fused launch."""
    pbufs, gbufs = [], []
    rank = None if ctx.mode == "distributed" else 0
    for p in params:
        pb = ctx.alloc(list(p.shape), torch.float32)
        gb = ctx.alloc(list(p.shape), grad_dtype)
        view = ctx.view(pb, rank)
        view.copy_(p.data.float())
        p.data = view
        g = ctx.view(gb, rank)
        g.zero_()
        p.grad = g if grad_dtype == torch.float32 else torch.zeros_like(view)
        pbufs.append(pb)
        gbufs.append(gb)
    return pbufs, gbufs


class _FusedBase(torch.optim.Optimizer):
    def __init__(self, params, defaults, ctx: Context, grad_dtype, bucket_cap):
        super().__init__(params, defaults)
        self.ctx = ctx
        self.plist = [p for g in self.param_groups for p in g["params"]]
        if len(self.param_groups) != 1:
            raise ValueError("one parameter group (the fused step applies one set of hyper-parameters)")
        for p in self.plist:
            if p.dtype != torch.float32:
                raise ValueError("master weights must be fp32")
        if grad_dtype not in (torch.float32, torch.float16, torch.bfloat16):
            raise ValueError("grad_dtype must be float32, float16 or bfloat16")
        self.grad_dtype = grad_dtype
        self.pbufs, self.gbufs = _rehome(ctx, self.plist, grad_dtype)
        self.tl = TensorList(ctx, [p.numel() for p in self.plist], bucket_cap=bucket_cap)
        self.m = ctx.alloc([self.tl.shard_elems], torch.float32)
        self.v = ctx.alloc([self.tl.shard_elems], torch.float32)
        for r in ctx.local_ranks():
            ctx.view(self.m, r).zero_()
            ctx.view(self.v, r).zero_()
        self.t = 0

    def zero_grad(self, set_to_none: bool = False):
        # the grads are heap views the kernels read (or their fp32 staging
        # tensors): keep them, zero in place
        for p in self.plist:
            p.grad.zero_()

    def _stage_grads(self):
        """16-bit grad_dtype: cast each fp32 .grad into its heap buffer."""
        if self.grad_dtype == torch.float32:
            return
        rank = None if self.ctx.mode == "distributed" else 0
        for p, gb in zip(self.plist, self.gbufs):
            self.ctx.view(gb, rank).copy_(p.grad)


class FusedAdam(_FusedBase):
    """Adam (torch.optim.Adam semantics, weight_decay 0) fused with the
    gradient all-reduce."""

    def __init__(self, params, ctx: Context, lr=1e-3, betas=(0.9, 0.999), eps=1e-8,
                 grad_dtype=torch.float32, math=_lib.MATH_FAST, bucket_cap=16384):
        super().__init__(params, dict(lr=lr, betas=betas, eps=eps), ctx, grad_dtype, bucket_cap)
        self.math = math

    @torch.no_grad()
    def step(self, closure=None):
        loss = closure() if closure is not None else None
        g = self.param_groups[0]
        self.t += 1
        hp = AdamHParams(lr=g["lr"], beta1=g["betas"][0], beta2=g["betas"][1], t=float(self.t), eps=g["eps"],
                         cv_beta1=False, math=self.math, algo=_lib.ALGO_TWO_SHOT)
        self._stage_grads()
        fused_rs_adam_ag(self.ctx, self.tl, self.gbufs, self.pbufs, self.m, self.v, hp)
        return loss


class FusedLAMB(_FusedBase):
    """LAMB with per-tensor trust ratio, fused with the gradient all-reduce."""

    def __init__(self, params, ctx: Context, lr=1e-3, betas=(0.9, 0.999), eps=1e-6, weight_decay=0.01,
                 grad_dtype=torch.float32, bucket_cap=16384):
        super().__init__(params, dict(lr=lr, betas=betas, eps=eps, weight_decay=weight_decay), ctx,
                         grad_dtype, bucket_cap)

    @torch.no_grad()
    def step(self, closure=None):
        loss = closure() if closure is not None else None
        g = self.param_groups[0]
        self.t += 1
        # trust_guard: a zero-norm tensor (e.g. a zero-initialised bias) steps
        # with ratio = lr instead of freezing or turning NaN (apex / NVLAMB)
        hp = LambHParams(lr=g["lr"], beta1=g["betas"][0], beta2=g["betas"][1], t=float(self.t), eps=g["eps"],
                         wd=g["weight_decay"], trust_guard=True)
        self._stage_grads()
        fused_rs_lamb_ag(self.ctx, self.tl, self.gbufs, self.pbufs, self.m, self.v, hp)
        return loss
