"""GPU: the torch.optim integration. A model's parameters and
grads live in the symmetric heap, backward() writes the grads the fused
kernel pulls, and step() matches torch.optim.Adam / a textbook LAMB."""
import pytest
import torch

from paper_2105_05720_b200.optim import FusedAdam, FusedLAMB
from paper_2105_05720_b200.runtime import Context

pytestmark = pytest.mark.gpu


def _model(seed):
    torch.manual_seed(seed)
    return torch.nn.Sequential(torch.nn.Linear(37, 64), torch.nn.GELU(), torch.nn.Linear(64, 5)).cuda()


def _batch(i):
    g = torch.Generator(device="cuda").manual_seed(100 + i)
    return torch.randn(16, 37, device="cuda", generator=g), torch.randn(16, 5, device="cuda", generator=g)


def test_fused_adam_matches_torch_adam():
    ctx = Context(1, heap_bytes=64 << 20)
    a, b = _model(0), _model(0)
    opt = FusedAdam(a.parameters(), ctx, lr=1e-2)
    ref = torch.optim.Adam(b.parameters(), lr=1e-2, eps=1e-8)
    for i in range(4):
        x, y = _batch(i)
        for m, o in ((a, opt), (b, ref)):
            o.zero_grad()
            torch.nn.functional.mse_loss(m(x), y).backward()
            o.step()
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert (pa - pb).abs().max().item() <= 1e-5 * pb.abs().max().item() + 1e-7
    ctx.close()


def _lamb_reference(params, state, lr, b1, b2, eps, wd, t):
    for p in params:
        st = state.setdefault(p, {"m": torch.zeros_like(p), "v": torch.zeros_like(p)})
        g = p.grad
        st["m"].mul_(b1).add_((1 - b1) * g)
        st["v"].mul_(b2).add_((1 - b2) * g * g)
        u = (st["m"] / (1 - b1 ** t)) / ((st["v"] / (1 - b2 ** t)).sqrt() + eps) + wd * p
        pn, un = p.norm(), u.norm()
        ratio = pn / un if pn > 0 and un > 0 else 1.0  # zero norm: step with lr (apex / NVLAMB)
        p.sub_(lr * ratio * u)


def test_fused_lamb_matches_reference_lamb():
    ctx = Context(1, heap_bytes=64 << 20)
    a, b = _model(1), _model(1)
    opt = FusedLAMB(a.parameters(), ctx, lr=1e-2, weight_decay=0.01)
    state = {}
    for i in range(3):
        x, y = _batch(i)
        opt.zero_grad()
        torch.nn.functional.mse_loss(a(x), y).backward()
        opt.step()
        for p in b.parameters():
            p.grad = None
        torch.nn.functional.mse_loss(b(x), y).backward()
        with torch.no_grad():
            _lamb_reference(list(b.parameters()), state, 1e-2, 0.9, 0.999, 1e-6, 0.01, i + 1)
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert (pa - pb).abs().max().item() <= 1e-5 * pb.abs().max().item() + 1e-7
    ctx.close()


def _zero_bias_model(seed):
    m = _model(seed)
    with torch.no_grad():
        for layer in (m[0], m[2]):
            layer.bias.zero_()
    return m


@pytest.mark.parametrize("grad_dtype", [torch.float32, torch.float16, torch.bfloat16])
def test_fused_lamb_zero_init_bias_and_grad_dtype(grad_dtype):
    """Zero-initialised biases (P = 0) step with ratio = lr instead of
    freezing or going NaN, and a 16-bit grad_dtype works: .grad stays fp32 for
    autograd and is cast into the 16-bit heap buffer the kernel pulls."""
    ctx = Context(1, heap_bytes=64 << 20)
    a, b = _zero_bias_model(2), _zero_bias_model(2)
    opt = FusedLAMB(a.parameters(), ctx, lr=1e-2, weight_decay=0.01, grad_dtype=grad_dtype)
    state = {}
    for i in range(3):
        x, y = _batch(i)
        opt.zero_grad()
        torch.nn.functional.mse_loss(a(x), y).backward()
        opt.step()
        for p in b.parameters():
            p.grad = None
        torch.nn.functional.mse_loss(b(x), y).backward()
        with torch.no_grad():
            for p in b.parameters():  # the kernel sees the grads at grad_dtype precision
                p.grad.copy_(p.grad.to(grad_dtype).float())
            _lamb_reference(list(b.parameters()), state, 1e-2, 0.9, 0.999, 1e-6, 0.01, i + 1)
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert torch.isfinite(pa).all()
        assert (pa - pb).abs().max().item() <= 1e-5 * pb.abs().max().item() + 1e-7
    assert a[0].bias.abs().max().item() > 0  # the zero bias moved
    ctx.close()


@pytest.mark.parametrize("grad_dtype", [torch.float16, torch.bfloat16])
def test_fused_adam_16bit_grad_dtype(grad_dtype):
    ctx = Context(1, heap_bytes=64 << 20)
    a, b = _model(3), _model(3)
    opt = FusedAdam(a.parameters(), ctx, lr=1e-2, grad_dtype=grad_dtype)
    ref = torch.optim.Adam(b.parameters(), lr=1e-2, eps=1e-8)
    for i in range(3):
        x, y = _batch(i)
        opt.zero_grad()
        torch.nn.functional.mse_loss(a(x), y).backward()
        opt.step()
        ref.zero_grad()
        torch.nn.functional.mse_loss(b(x), y).backward()
        with torch.no_grad():
            for p in b.parameters():
                p.grad.copy_(p.grad.to(grad_dtype).float())
        ref.step()
    # 16-bit grads put some elements in Adam's eps-dominated regime (sqrt(v)
    # ~ eps), where torch's sqrt(v)/sqrt(bc2) + eps and the kernel's
    # sqrt(v/bc2) + eps round apart by a few e-6 of |p|
    for pa, pb in zip(a.parameters(), b.parameters()):
        assert (pa - pb).abs().max().item() <= 3e-5 * pb.abs().max().item() + 1e-7
    ctx.close()
