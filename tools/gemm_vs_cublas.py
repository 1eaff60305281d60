"""C3 GEMM shape [8192x384] x [384x3072] bf16: our tcgen05 kernel (coconet_matmul,
8 virtual ranks and 1 rank) next to cuBLAS (torch.matmul, one and batched x8)
on the same GPU. Probe only. Usage: python tools/gemm_vs_cublas.py"""
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))

from paper_2105_05720_b200 import _lib  # noqa: E402
from paper_2105_05720_b200.collectives import matmul  # noqa: E402
from paper_2105_05720_b200.runtime import Context  # noqa: E402
from tools.pattern_probe import timeit  # noqa: E402

M, K, N = 8192, 384, 3072
flops = 2.0 * M * N * K
out = {}
a = torch.randn(8, M, K, device="cuda", dtype=torch.bfloat16)
b = torch.randn(8, K, N, device="cuda", dtype=torch.bfloat16) * K ** -0.5
ms = timeit(lambda: torch.matmul(a[0], b[0]), 50)
out["cublas_1_us"] = ms * 1e3
out["cublas_1_tflops"] = flops / ms / 1e9
ms = timeit(lambda: torch.bmm(a, b), 20)
out["cublas_bmm8_us"] = ms * 1e3
out["cublas_bmm8_tflops"] = 8 * flops / ms / 1e9
for W in (1, 8):
    ctx = Context(W, heap_bytes=(W * 0 + 1) << 30)
    x, w, c = ctx.alloc([M, K], torch.bfloat16), ctx.alloc([K, N], torch.bfloat16), ctx.alloc([M, N], torch.bfloat16)
    for r in range(W):
        ctx.view(x, r).copy_(a[r % 8])
        ctx.view(w, r).copy_(b[r % 8])
    ms = timeit(lambda: matmul(ctx, x, w, c, math=_lib.MATH_FAST), 20)
    out[f"coconet_{W}ranks_us"] = ms * 1e3
    out[f"coconet_{W}ranks_tflops"] = W * flops / ms / 1e9
    err = (ctx.view(c, 0).float() - torch.matmul(a[0].float(), b[0].float())).abs().max().item()
    out[f"coconet_{W}ranks_maxabs_err"] = err
    ctx.close()
print(json.dumps(out, indent=1))
