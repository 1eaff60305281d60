"""Symmetric heap through the C ABI: free/reuse of offsets, and symmetric
buffers freed and reallocated keep working for collectives."""
import pytest
import torch

from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import TensorList, allreduce
from tests.dp_util import new_ctx

pytestmark = pytest.mark.gpu


def test_alloc_free_reuse():
    ctx = new_ctx(2, heap_mb=16)
    a = ctx.alloc([1000])
    b = ctx.alloc([5000])
    c = ctx.alloc([10])
    assert a.offset < b.offset < c.offset
    ctx.free(b)
    d = ctx.alloc([4000])          # first fit: lands where b was
    assert d.offset == b.offset
    ctx.free(d)
    with pytest.raises(_lib.CoconetError) as e:
        ctx.free(d)                # double free is rejected
    assert e.value.name == "InvalidInput"
    high = ctx.high_water()
    assert high >= c.offset + 256
    ctx.reset()
    e = ctx.alloc([10])
    assert e.offset == a.offset
    ctx.close()


def test_freed_buffers_still_serve_collectives():
    W, n = 4, 3000
    ctx = new_ctx(W, heap_mb=16)
    tmp = [ctx.alloc([n]) for _ in range(3)]
    for t in tmp:
        ctx.free(t)
    x, out = ctx.alloc([n]), ctx.alloc([n])
    assert x.offset == tmp[0].offset
    tl = TensorList(ctx, [n])
    for r in range(W):
        ctx.view(x, r).fill_(float(r + 1))
    allreduce(ctx, tl, [x], [out])
    ctx.check()
    for r in range(W):
        assert torch.all(ctx.view(out, r) == 10.0)
    ctx.close()


def test_oom_reports_largest_free_block():
    ctx = new_ctx(1, heap_mb=4)
    with pytest.raises(_lib.CoconetError) as e:
        ctx.alloc([64 << 20])
    assert e.value.name == "OutOfHeap" and "largest free block" in str(e.value)
    ctx.close()
