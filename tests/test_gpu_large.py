"""Maximum sizes: a single tensor of more than 2^31 elements through the
fused RS-Adam-AG (C5 is 3.9e9 parameters: "64-bit indexing
required"). The kernels' element, quad and byte offsets all cross 2^31 here.

Checked bit for bit (EXACT math) against the oracle's restatement
(oracle/coconet_oracle.py adam_exact, state.hpp/expr.hpp semantics) on a
sample of elements: random ones, the last 64 and those around 2^31. m and v
start at zero, so the expected update depends only on g and p, which are read
back at the sampled indices."""
import numpy as np
import pytest
import torch

from oracle import coconet_oracle as co
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import (AdamHParams, LambHParams, TensorList, fused_rs_adam_ag,
                                               fused_rs_lamb_ag, gen_values)
from paper_2105_05720_b200.runtime import Context

pytestmark = pytest.mark.gpu

N = (1 << 31) + 1029


def _sample(n):
    rng = np.random.default_rng(7)
    idx = np.concatenate([rng.integers(0, n, 4096), np.arange(n - 64, n), np.arange((1 << 31) - 32, (1 << 31) + 32)])
    return torch.from_numpy(np.unique(idx)).cuda()


@pytest.mark.parametrize("W,cap", [(1, 16384), (2, 1024)])
def test_adam_beyond_2_pow_31_elements(W, cap):
    if torch.cuda.get_device_properties(0).total_memory < (W * 26 + 8) << 30:
        pytest.skip("needs the B200's HBM")
    ctx = Context(W, heap_bytes=N * 4 * 2 + (N // W + 4096) * 4 * 2 + (64 << 20), timeout_ms=20000)
    try:
        tl = TensorList(ctx, [N], bucket_cap=cap)
        g, p = ctx.alloc([N]), ctx.alloc([N])
        m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
        for r in range(W):
            gen_values(ctx, ctx.view(g, r), 1, "g", "local", r, [N], group_size=W)
            gen_values(ctx, ctx.view(p, r), 1, "p", "replicated", r, [N], group_size=W)
            ctx.view(m, r).zero_()
            ctx.view(v, r).zero_()
        idx = _sample(N)
        gs = np.stack([ctx.view(g, r)[idx].cpu().numpy() for r in range(W)])
        p0 = ctx.view(p, 0)[idx].cpu().numpy()
        hp = AdamHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=3.0, math=_lib.MATH_EXACT, algo=_lib.ALGO_TWO_SHOT)
        fused_rs_adam_ag(ctx, tl, [g], [p], m, v, hp)
        ctx.check()
        # one tensor: bucket order is element order, so the owner of element i
        # is the flat chunk that holds i; the fold is the ring order from owner+1
        bounds = np.asarray(co.flat_chunks(N, W)[1:])
        owner = np.searchsorted(bounds, idx.cpu().numpy(), side="right")
        gred = co.ring_reduce(gs, owner)
        k = co.adam_consts(1e-3, 0.9, 0.999, 3.0)
        zeros = np.zeros_like(p0)
        _, _, want = co.adam_exact(gred, zeros, zeros, p0, k)
        for r in range(W):
            got = ctx.view(p, r)[idx].cpu().numpy()
            bad = np.flatnonzero(got.view(np.uint32) != want.view(np.uint32))
            assert bad.size == 0, (r, idx[bad[:5]].tolist(), got[bad[:5]], want[bad[:5]])
    finally:
        ctx.close()


def test_lamb_beyond_2_pow_31_elements():
    """The headline LAMB path (TMA schedule, fp16 grads) on one tensor of more
    than 2^31 elements: the per-tensor norms are sums over all of it. The
    expected trust ratio is summed in fp64 by torch in chunks; the update is
    compared at the sampled elements within the north star's 1e-5."""
    if torch.cuda.get_device_properties(0).total_memory < (40 << 30):
        pytest.skip("needs the B200's HBM")
    ctx = Context(1, heap_bytes=N * 14 + (64 << 20), timeout_ms=20000)
    try:
        tl = TensorList(ctx, [N], bucket_cap=16384)
        g, p = ctx.alloc([N], torch.float16), ctx.alloc([N])
        m, v = ctx.alloc([tl.shard_elems]), ctx.alloc([tl.shard_elems])
        gen_values(ctx, ctx.view(g, 0), 1, "g", "local", 0, [N], group_size=1)
        gen_values(ctx, ctx.view(p, 0), 1, "p", "replicated", 0, [N], group_size=1)
        ctx.view(m, 0).zero_()
        ctx.view(v, 0).zero_()
        k = co.lamb_consts(1e-3, 0.9, 0.999, 1.0, 1e-6, 0.01)
        gv, pv = ctx.view(g, 0), ctx.view(p, 0)

        def u_of(gc, pc):
            gc, pc = gc.double(), pc.double()
            mn = k["c1"] * gc
            vn = (k["c2"] * gc) * gc
            return (mn / k["bc1"]) / (torch.sqrt(vn / k["bc2"]) + k["eps"]) + k["wd"] * pc

        P = U = 0.0
        step = 1 << 28
        for s in range(0, N, step):
            gc, pc = gv[s:s + step], pv[s:s + step]
            P += float((pc.double() ** 2).sum())
            U += float((u_of(gc, pc) ** 2).sum())
        idx = _sample(N)
        u = u_of(gv[idx], pv[idx])
        p0 = pv[idx].double()
        step_want = ((k["lr"] * np.sqrt(P) / np.sqrt(U)) * u).cpu().numpy()
        want = (p0 - (k["lr"] * np.sqrt(P) / np.sqrt(U)) * u).float().cpu().numpy()
        p0 = p0.cpu().numpy()
        hp = LambHParams(lr=1e-3, beta1=0.9, beta2=0.999, t=1.0, eps=1e-6, wd=0.01)
        fused_rs_lamb_ag(ctx, tl, [g], [p], m, v, hp)
        ctx.check()
        got = pv[idx].cpu().numpy()
        assert co.max_rel_deviation(got, want) <= 1e-5
        # the step itself (lr x trust ratio x u, ~5e-4) to 1e-3: an fp32 p
        # carries it to ~1e-4, so a wrong norm anywhere in 2^31 elements shows
        assert co.max_rel_deviation(p0 - got.astype(np.float64), step_want) <= 1e-3
    finally:
        ctx.close()
