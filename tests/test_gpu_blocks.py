"""Block-level integration: affine merge + MS norms +
ReGELU2 / ReSwiGLU2 inside ViT / LLaMA FFN half-blocks.  The forward is
unchanged, the memory-sharing backward is exact, and the
activation memory kept for backward matches the analytic count byte for byte."""
import pytest
import torch

import synth
import paper_2406_16282_b200 as P
from paper_2406_16282_b200.blocks import LlamaMLP, ViTMLP, activation_bytes

pytestmark = pytest.mark.gpu
DEV = "cuda"


def rel(a, b):
    return float((a.float() - b.float()).norm() / b.float().norm())


@pytest.mark.parametrize("cls,c,h", [(ViTMLP, 768, 3072), (LlamaMLP, 512, 1376)])
def test_forward_unchanged_and_ms_backward_exact(cls, c, h):
    torch.manual_seed(0)
    blk = cls(c, h, device=DEV)
    x = synth.norm_input(256, c, "bf16").to(DEV)
    ours_ms = blk.to_ours(act=False)          # merge + MS norm only: exact gradients
    ours = blk.to_ours()                      # + ReGELU2 / ReSwiGLU2
    xs = [x.clone().requires_grad_(True) for _ in range(3)]
    outs = [m(xi) for m, xi in zip((blk, ours_ms, ours), xs)]
    assert rel(outs[1], outs[0]) < 1e-2 and rel(outs[2], outs[0]) < 1e-2
    dy = synth.grad_input(256, c, "bf16").to(DEV)
    for o in outs:
        o.backward(dy)
    assert rel(xs[1].grad, xs[0].grad) < 2e-2                 # MS backward == exact backward
    assert 0 < rel(xs[2].grad, xs[0].grad) < 0.6              # Approx-BP: close, not equal


def test_vit_block_saved_bytes():
    R, c, h = 64 * 197 // 8, 768, 3072
    blk = ViTMLP(c, h, device=DEV)
    x = synth.norm_input(R, c, "bf16").to(DEV).requires_grad_(True)
    exact = activation_bytes(blk, x)
    ours = activation_bytes(blk.to_ours(), x)
    assert ours == R * c * 2 + 4 * R + P.codes_bytes(R * h) + R * h * 2      # y(shared) + rstd + codes + fc2 in
    unit = R * c * 2
    assert exact / unit >= 10.9 and ours / unit <= 5.51                       # 11 -> 5.5 units (App. B)


def test_llama_block_saved_bytes():
    R, c, h = 512, 4096, 11008
    blk = LlamaMLP(c, h, device=DEV)
    x = synth.norm_input(R, c, "bf16").to(DEV).requires_grad_(True)
    exact = activation_bytes(blk, x)
    ours = activation_bytes(blk.to_ours(), x)
    assert ours == R * c * 2 + 4 * R + 3 * R * h * 2 + P.codes_bytes(R * h)  # y + rstd + up, a, h + codes
    assert exact > ours + 2 * R * c                                          # fp32 norm input and SiLU input gone
