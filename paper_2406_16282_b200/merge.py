"""Affine merge for memory-sharing normalisation.

MS-LN / MS-RMSNorm are parameter-free: the affine (alpha, beta) of LayerNorm /
RMSNorm is folded into the linear layer(s) that consume the normalised output
(App. F):

    W~ = W diag(alpha),   b~ = W beta + b        (LayerNorm)
    W~ = W diag(alpha),   b~ = b                 (RMSNorm, beta = 0)

so that  W~ MSLN(x) + b~ == W LN(x; alpha, beta) + b  exactly in real
arithmetic.  This is one-time weight preparation (a plain matmul), not part
of the per-step hot path, so it uses torch ops.  Under QLoRA the paper merges
into the transposed NF4 weight to keep the block-wise quantisation
 -- out of scope here (no NF4 storage).
"""
from __future__ import annotations

import torch

from .modules import MSLayerNorm, MSRMSNorm


@torch.no_grad()
def merge_ln(weight: torch.Tensor, bias, alpha: torch.Tensor, beta) -> tuple:
    """(W~, b~) = (W diag(alpha), W beta + b).  weight: [out, p]."""
    if weight.shape[-1] != alpha.numel():
        raise ValueError("dimension mismatch: W is [out, p], alpha is [p]")
    wd = weight.double()
    w_new = (wd * alpha.double()[None, :]).to(weight.dtype)
    b_new = None
    if beta is not None or bias is not None:
        b = torch.zeros(weight.shape[0], dtype=torch.float64, device=weight.device)
        if beta is not None:
            b = b + wd @ beta.double()
        if bias is not None:
            b = b + bias.double()
        b_new = b.to(weight.dtype)
    return w_new, b_new


@torch.no_grad()
def merge_rms(weight: torch.Tensor, bias, alpha: torch.Tensor) -> tuple:
    """(W~, b~) = (W diag(alpha), b)."""
    return merge_ln(weight, bias, alpha, None)


@torch.no_grad()
def fold_norm_into_linears(norm: torch.nn.Module, linears, eps=None):
    """Replace a LayerNorm / RMSNorm (with affine) feeding `linears` by the
    parameter-free MS variant, folding its affine into every consumer linear
    in place.  Returns the MS module.  Works for torch.nn.LayerNorm and any
    RMSNorm-like module exposing .weight (and .eps / .variance_epsilon)."""
    linears = list(linears)
    is_ln = isinstance(norm, torch.nn.LayerNorm)
    alpha = norm.weight if getattr(norm, "weight", None) is not None else None
    beta = getattr(norm, "bias", None) if is_ln else None
    p = alpha.numel() if alpha is not None else linears[0].in_features
    if alpha is None:
        alpha = torch.ones(p, device=linears[0].weight.device)
    for lin in linears:
        w, b = merge_ln(lin.weight, lin.bias, alpha, beta)
        lin.weight.copy_(w)
        if b is not None:
            if lin.bias is None:
                lin.bias = torch.nn.Parameter(b)
            else:
                lin.bias.copy_(b)
    if eps is None:
        eps = getattr(norm, "eps", None) or getattr(norm, "variance_epsilon", 1e-6)
    return (MSLayerNorm if is_ln else MSRMSNorm)(p, eps)
