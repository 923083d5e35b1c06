"""Transformer sub-blocks built from the MS / Re modules, for measuring the
activation memory the method saves at block level (
the paper's Fig. 2 composition).

* ``ViTMLP``:  x + fc2(act(fc1(norm(x))))      -- ViT / RoBERTa FFN half-block
* ``LlamaMLP``: x + down(silu(gate(n)) * up(n)), n = norm(x)  -- LLaMA FFN half-block

``exact=True`` builds the reference composition the paper compares against:
LayerNorm / RMSNorm with affine computed in fp32 (AMP keeps norms in fp32,
P:L816), exact GELU / SiLU, unmerged linears.  ``exact=False`` builds
ours: the affine folded into the consumer linears (merge.py), MS-LN / MS-RMSNorm,
ReGELU2 / fused ReSwiGLU2.  Both run the same weights, so their outputs agree
to bf16 rounding and their saved activations can be compared byte for byte.
"""
from __future__ import annotations

import copy

import torch

from . import modules
from .merge import fold_norm_into_linears


class RMSNormRef(torch.nn.Module):
    """The textbook RMSNorm with affine, in fp32 (reference only)."""

    def __init__(self, p, eps=1e-6, device=None):
        super().__init__()
        self.weight = torch.nn.Parameter(torch.ones(p, device=device))
        self.eps = eps

    def forward(self, x):
        xf = x.float()
        y = xf * torch.rsqrt(xf.pow(2).mean(-1, keepdim=True) + self.eps)
        return (self.weight * y).to(x.dtype)


class LayerNormRef(torch.nn.LayerNorm):
    """torch LayerNorm with affine, evaluated in fp32 as under AMP."""

    def forward(self, x):
        return super().forward(x.float()).to(x.dtype)


class ViTMLP(torch.nn.Module):
    def __init__(self, c=768, hidden=3072, eps=1e-6, dtype=torch.bfloat16, device="cuda", seed=0):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.norm = LayerNormRef(c, eps=eps, device=device)
        with torch.no_grad():
            self.norm.weight.copy_(1 + 0.1 * torch.randn(c, generator=g))
            self.norm.bias.copy_(0.1 * torch.randn(c, generator=g))
        self.fc1 = torch.nn.Linear(c, hidden, device=device, dtype=dtype)
        self.fc2 = torch.nn.Linear(hidden, c, device=device, dtype=dtype)
        self.act = torch.nn.GELU()
        self.exact = True

    def to_ours(self, act=True):
        """MS-LN with the affine folded into fc1; ReGELU2 unless act=False
        (act=False isolates the exact memory-sharing part for gradient checks)."""
        m = copy.deepcopy(self)
        m.norm = fold_norm_into_linears(m.norm, [m.fc1])
        if act:
            m.act = modules.ReGELU2()
        m.exact = False
        return m

    def forward(self, x):
        return x + self.fc2(self.act(self.fc1(self.norm(x))))


class LlamaMLP(torch.nn.Module):
    def __init__(self, c=4096, hidden=11008, eps=1e-6, dtype=torch.bfloat16, device="cuda", seed=0):
        super().__init__()
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.norm = RMSNormRef(c, eps=eps, device=device)
        with torch.no_grad():
            self.norm.weight.copy_(1 + 0.1 * torch.randn(c, generator=g))
        self.gate = torch.nn.Linear(c, hidden, bias=False, device=device, dtype=dtype)
        self.up = torch.nn.Linear(c, hidden, bias=False, device=device, dtype=dtype)
        self.down = torch.nn.Linear(hidden, c, bias=False, device=device, dtype=dtype)
        self.exact = True

    def to_ours(self, act=True):
        m = copy.deepcopy(self)
        m.norm = fold_norm_into_linears(m.norm, [m.gate, m.up])
        m.exact = False
        m.fused_act = act
        return m

    def forward(self, x):
        n = self.norm(x)
        if self.exact or not getattr(self, "fused_act", True):
            h = torch.nn.functional.silu(self.gate(n)) * self.up(n)
        else:
            h = modules.ReSwiGLU2Fn.apply(self.gate(n), self.up(n))
        return x + self.down(h)


def activation_bytes(block: torch.nn.Module, x: torch.Tensor) -> int:
    """Activation bytes `block(x)` keeps for backward, deduplicated by storage,
    excluding parameters (weights are not activations)."""
    params = {p.untyped_storage().data_ptr() for p in block.parameters()}
    seen = {}

    def pack(t):
        st = t.untyped_storage()
        if st.data_ptr() not in params:
            seen[st.data_ptr()] = st.nbytes()
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = block(x)
    del out
    return int(sum(seen.values()))
