"""Reduce / Broadcast kernels (runtime.hpp:415-436) at the C-ABI level,
against a numpy restatement of the Engine's semantics: rank-order fp32 fold
on the root, zeros elsewhere; broadcast copies the root's tensor."""
import numpy as np
import pytest
import torch

from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import broadcast, reduce
from tests.dp_util import new_ctx

pytestmark = pytest.mark.gpu

RED = {_lib.SUM: np.add, _lib.MAX: np.maximum, _lib.MIN: np.minimum}


@pytest.mark.parametrize("W", [1, 2, 3, 4, 8])
@pytest.mark.parametrize("n", [1, 7, 4096, 100_003])
@pytest.mark.parametrize("red", [_lib.SUM, _lib.MAX, _lib.MIN])
def test_reduce_rank_order(W, n, red):
    rng = np.random.default_rng(W * 1000 + n + red)
    xs = rng.uniform(-1, 1, (W, n)).astype(np.float32)
    root = W - 1
    ctx = new_ctx(W)
    x, out = ctx.alloc([n]), ctx.alloc([n])
    for r in range(W):
        ctx.view(x, r).copy_(torch.from_numpy(xs[r]))
        ctx.view(out, r).fill_(7.0)
    reduce(ctx, x, out, root=root, reducer=red)
    ctx.check()
    acc = xs[0].copy()
    for r in range(1, W):
        acc = RED[red](acc, xs[r]).astype(np.float32)  # fp32 fold in rank order
    for r in range(W):
        got = ctx.view(out, r).cpu().numpy()
        assert np.array_equal(got, acc if r == root else np.zeros(n, np.float32))
    ctx.close()


@pytest.mark.parametrize("W", [2, 4, 8])
def test_reduce_in_place_many_ctas(W):
    """x aliases out over a multi-CTA grid: a non-root CTA zeroes only the
    vectors the root's CTA of the same index has finished reading."""
    n = 1 << 22
    rng = np.random.default_rng(W)
    xs = rng.uniform(-1, 1, (W, n)).astype(np.float32)
    ctx = new_ctx(W)
    x = ctx.alloc([n])
    for r in range(W):
        ctx.view(x, r).copy_(torch.from_numpy(xs[r]))
    root = 1
    reduce(ctx, x, x, root=root)
    ctx.check()
    acc = xs[0].copy()
    for r in range(1, W):
        acc = (acc + xs[r]).astype(np.float32)
    for r in range(W):
        got = ctx.view(x, r).cpu().numpy()
        assert np.array_equal(got, acc if r == root else np.zeros(n, np.float32)), r
    ctx.close()


def test_reduce_in_place_and_bf16():
    W, n = 4, 4096
    ctx = new_ctx(W)
    x = ctx.alloc([n], torch.bfloat16)
    for r in range(W):
        ctx.view(x, r).fill_(float(r + 1))
    reduce(ctx, x, x, root=2)
    ctx.check()
    assert ctx.view(x, 2).float().cpu().tolist() == [10.0] * n
    for r in (0, 1, 3):
        assert ctx.view(x, r).float().abs().sum().item() == 0.0
    ctx.close()


@pytest.mark.parametrize("W", [1, 2, 4, 8])
@pytest.mark.parametrize("n", [3, 4096, 65_537])
@pytest.mark.parametrize("dtype", [torch.float32, torch.float16])
def test_broadcast(W, n, dtype):
    ctx = new_ctx(W)
    x, out = ctx.alloc([n], dtype), ctx.alloc([n], dtype)
    for r in range(W):
        ctx.view(x, r).uniform_(-1, 1)
    root = W // 2
    want = ctx.view(x, root).cpu().clone()
    broadcast(ctx, x, out, root=root)
    ctx.check()
    for r in range(W):
        assert torch.equal(ctx.view(out, r).cpu(), want)
    broadcast(ctx, x, x, root=root)  # in place: the root's x reaches every rank
    ctx.check()
    for r in range(W):
        assert torch.equal(ctx.view(x, r).cpu(), want)
    ctx.close()


def test_rooted_errors():
    ctx = new_ctx(2)
    x = ctx.alloc([8])
    with pytest.raises(_lib.CoconetError) as e:
        reduce(ctx, x, x, root=2)
    assert e.value.name == "NoSuchRank"
    with pytest.raises(_lib.CoconetError):
        broadcast(ctx, x, x, root=-1)
    ctx.close()
