"""GPU: the MatMul of the model-parallel pattern (eval_matmul, state.hpp:94-121)
on tcgen05 (FAST, bf16/fp16 in, fp32 accumulate) against a plain torch fp32
reference, the EXACT fp64 path bit-for-bit against the restated eval_matmul,
and the overlapped MatMul + fused AllReduce epilogue (mp_overlap.json)
against the sequential composition and the reference's golden digest."""
import numpy as np
import pytest
import torch

from oracle import coconet_oracle as co
from paper_2105_05720_b200 import _lib
from paper_2105_05720_b200.collectives import BdrHParams, fused_rs_bdr_ag, matmul, mm_overlap_fused_ar
from tests.dp_util import golden, new_ctx
from tests.test_gpu_mp_pp import mp_inputs

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 128, 64), (256, 384, 128), (512, 768, 384), (1024, 3072, 384),
                                   (384, 256, 256)])
@pytest.mark.parametrize("dtype", [torch.bfloat16, torch.float16])
@pytest.mark.parametrize("W", [1, 2])
def test_tcgen05_matmul_vs_torch_fp32(M, N, K, dtype, W):
    torch.manual_seed(M + N + K)
    ctx = new_ctx(W, heap_mb=128)
    a, b = ctx.alloc([M, K], dtype), ctx.alloc([K, N], dtype)
    c = ctx.alloc([M, N], torch.float32)
    refs = []
    for r in range(W):
        ctx.view(a, r).copy_(torch.randn(M, K).to(dtype))
        ctx.view(b, r).copy_(torch.randn(K, N).to(dtype))
        refs.append(ctx.view(a, r).float() @ ctx.view(b, r).float())
    matmul(ctx, a, b, c, math=_lib.MATH_FAST)
    ctx.check()
    for r in range(W):
        got = ctx.view(c, r)
        err = (got - refs[r]).abs().max().item() / refs[r].abs().max().item()
        assert err < 1e-3, (r, err)


@pytest.mark.parametrize("M,N,K", [(16, 64, 16), (100, 70, 33), (64, 128, 96)])
def test_exact_matmul_bitwise(M, N, K):
    rng = np.random.default_rng(M * N)
    x = rng.uniform(-1, 1, (M, K)).astype(np.float32)
    w = rng.uniform(-1, 1, (K, N)).astype(np.float32)
    ctx = new_ctx(1)
    a, b, c = ctx.alloc([M, K]), ctx.alloc([K, N]), ctx.alloc([M, N])
    ctx.view(a, 0).copy_(torch.from_numpy(x))
    ctx.view(b, 0).copy_(torch.from_numpy(w))
    matmul(ctx, a, b, c, math=_lib.MATH_EXACT)
    ctx.check()
    assert np.array_equal(ctx.view(c, 0).cpu().numpy(), co.matmul_exact(x, w))


@pytest.mark.parametrize("name", ["mp_W1_B2_S8_H64", "mp_W2_B2_S8_H64", "mp_W4_B2_S8_H64", "mp_W8_B2_S16_H128"])
def test_mp_program_end_to_end_exact_digest(name):
    """MatMul (EXACT, fp64) -> FusedAllReduce(dropout(layer + b) + r) entirely on
    the device reproduces the reference Engine's digest on mp_overlap.json."""
    rec = golden(name)
    W, rows, H, xs, ws, b, res = mp_inputs(rec)
    ctx = new_ctx(W)
    x, w = ctx.alloc([rows, H // W]), ctx.alloc([H // W, H])
    part, bb, rr, out = ctx.alloc([rows, H]), ctx.alloc([H]), ctx.alloc([rows, H]), ctx.alloc([rows, H])
    for r in range(W):
        ctx.view(x, r).copy_(torch.from_numpy(xs[r]))
        ctx.view(w, r).copy_(torch.from_numpy(ws[r]))
        ctx.view(bb, r).copy_(torch.from_numpy(b))
        ctx.view(rr, r).copy_(torch.from_numpy(res))
    matmul(ctx, x, w, part, math=_lib.MATH_EXACT)
    fused_rs_bdr_ag(ctx, part, bb, rr, out, BdrHParams(0.1, 1, co.fnv1a("dropout"), _lib.MATH_EXACT))
    ctx.check()
    got = ctx.view(out, 0).cpu().numpy().ravel()
    assert "%016x" % co.digest_results({"out0": [got]}) == rec["engine_sched_digest"]


@pytest.mark.parametrize("W,rows,H", [(1, 256, 512), (2, 512, 768), (4, 1024, 1536), (8, 1024, 3072),
                                       (4, 512, 512), (2, 256, 512), (2, 256, 1536), (4, 256, 2048)])
@pytest.mark.parametrize("mode", ["fused", "sequential", "auto"])
def test_mm_overlap_matches_sequential(W, rows, H, mode, monkeypatch):
    """OverlapGroup{MatMul, FusedAllReduce}. The tile-flag-overlapped pair
    (mode=fused) and the two kernels back to back give bit-identical output
    (Overlap.OutputBitIdenticalToSequential, test_overlap.cpp:35-43). AUTO is
    the all-gather -> GEMM kernel where the column block is a multiple of 128 wide
    (no partial products; the sum is accumulated in fp32 over the whole K;
    blocks wider than 384 columns run as 384/256/128-column sub-blocks):
    within 1e-2 of the fp32 reference for bf16 activations, the dropout mask
    bit-exact (dropped elements equal the residual), and the same output on
    every rank; other shapes fall back to the two kernels."""
    if mode == "auto":
        monkeypatch.delenv("COCONET_MP_OVERLAP", raising=False)
    else:
        monkeypatch.setenv("COCONET_MP_OVERLAP", mode)
    dtype = torch.bfloat16
    k = H // W
    torch.manual_seed(W * rows)
    ctx = new_ctx(W, heap_mb=256)
    x, w = ctx.alloc([rows, k], dtype), ctx.alloc([k, H], dtype)
    part, bb, rr = ctx.alloc([rows, H], dtype), ctx.alloc([H], dtype), ctx.alloc([rows, H], dtype)
    out1, out2 = ctx.alloc([rows, H], dtype), ctx.alloc([rows, H], dtype)
    bias = (torch.randn(H) * 0.1).to(dtype)
    resid = torch.randn(rows, H).to(dtype)
    for r in range(W):
        ctx.view(x, r).copy_(torch.randn(rows, k).to(dtype))
        ctx.view(w, r).copy_((torch.randn(k, H) / k ** 0.5).to(dtype))
        ctx.view(bb, r).copy_(bias)
        ctx.view(rr, r).copy_(resid)
    hp = BdrHParams(0.1, 5, co.fnv1a("dropout"), _lib.MATH_FAST)
    for _ in range(2):  # twice: flags/counters must be reusable across calls
        mm_overlap_fused_ar(ctx, x, w, bb, rr, part, out1, hp)
        ctx.check()
    matmul(ctx, x, w, part, math=_lib.MATH_FAST)
    fused_rs_bdr_ag(ctx, part, bb, rr, out2, hp)
    ctx.check()
    ag = mode == "auto" and W > 1 and (H // W) % 128 == 0 and rows % 256 == 0
    for r in range(W):
        if ag:
            assert torch.equal(ctx.view(out1, r), ctx.view(out1, 0)), r
        else:
            assert torch.equal(ctx.view(out1, r), ctx.view(out2, r)), r
    # fp32 reference of the whole layer
    full = sum(ctx.view(x, r).float() @ ctx.view(w, r).float() for r in range(W))
    keep = torch.from_numpy(co.dropout_keep(5, co.fnv1a("dropout"), np.arange(rows * H), 0.1).reshape(rows, H)).cuda()
    want = torch.where(keep, (full + bias.float().cuda()) / 0.9, torch.zeros_like(full)) + resid.float().cuda()
    got = ctx.view(out1, 0).float()
    assert ((got - want).abs().max() / want.abs().max()).item() < 1e-2
    # dropped elements are exactly the residual (the mask is the reference's)
    assert torch.equal(got[~keep], resid.float().cuda()[~keep])
