"""Affine merge on CPU, float64:
W~ MSLN(x) + b~ == W LN(x; alpha, beta) + b, and the parameter gradients
correspond through the merge map (dW~ = dW diag(alpha)) -- SPEC S:L286-295.
MS-LN / MS-RMSNorm are written out here with torch ops (the CUDA kernels need a
GPU; the merge itself is plain weight preparation)."""
import torch

from paper_2406_16282_b200.merge import merge_ln, merge_rms


def msln(x, eps):
    m = x.mean(-1, keepdim=True)
    return (x - m) / torch.sqrt(((x - m) ** 2).mean(-1, keepdim=True) + eps)


def msrms(x, eps):
    return x / torch.sqrt((x * x).mean(-1, keepdim=True) + eps)


def test_merge_ln_pipeline_equivalence_and_grad_map():
    g = torch.Generator().manual_seed(0)
    p, out, eps = 16, 5, 1e-6
    x = torch.randn(7, p, generator=g, dtype=torch.float64)
    alpha = 1 + 0.3 * torch.randn(p, generator=g, dtype=torch.float64)
    beta = 0.3 * torch.randn(p, generator=g, dtype=torch.float64)
    W = torch.randn(out, p, generator=g, dtype=torch.float64, requires_grad=True)
    b = torch.randn(out, generator=g, dtype=torch.float64)
    ref = torch.nn.functional.layer_norm(x, (p,), alpha, beta, eps) @ W.T + b
    Wt, bt = merge_ln(W.detach(), b, alpha, beta)
    Wt.requires_grad_(True)
    bt.requires_grad_(True)
    got = msln(x, eps) @ Wt.T + bt
    assert torch.allclose(got, ref, rtol=1e-12, atol=1e-12)
    dy = torch.randn(7, out, generator=g, dtype=torch.float64)
    ref.backward(dy)
    got.backward(dy)
    # chain rule through W~ = W diag(alpha), b~ = W beta + b:
    # dL/dW = dL/dW~ diag(alpha) + dL/db~ beta^T
    assert torch.allclose(W.grad, Wt.grad * alpha[None, :] + bt.grad[:, None] * beta[None, :], rtol=1e-10)
    # identity affine: no-op merge; W = I: W~ = diag(alpha), b~ = beta
    W2, b2 = merge_ln(W.detach(), b, torch.ones(p, dtype=torch.float64), torch.zeros(p, dtype=torch.float64))
    assert torch.equal(W2, W.detach()) and torch.allclose(b2, b)
    W3, b3 = merge_ln(torch.eye(p, dtype=torch.float64), None, alpha, beta)
    assert torch.allclose(W3, torch.diag(alpha)) and torch.allclose(b3, beta)


def test_merge_rms_pipeline_equivalence():
    g = torch.Generator().manual_seed(1)
    p, out, eps = 32, 3, 1e-6
    x = torch.randn(4, p, generator=g, dtype=torch.float64)
    alpha = 1 + 0.3 * torch.randn(p, generator=g, dtype=torch.float64)
    W = torch.randn(out, p, generator=g, dtype=torch.float64)
    ref = (alpha * msrms(x, eps)) @ W.T
    Wt, bt = merge_rms(W, None, alpha)
    assert bt is None
    assert torch.allclose(msrms(x, eps) @ Wt.T, ref, rtol=1e-12, atol=1e-12)
