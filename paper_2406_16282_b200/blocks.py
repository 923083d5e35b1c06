"""Whole transformer blocks built from the MS / Re modules, for measuring the
activation memory the method saves at block level under the paper's
fine-tuning regimes (Fig. 2 composition P:L214, Fig. 5 /
Fig. 6 unit model P:L816, decoded in SURVEY App. B).

* ``Block("vit", ...)``   pre-norm ViT / RoBERTa block:
      x = x + proj(attn(q(n1), k(n1), v(n1))),  n1 = LN1(x)
      x = x + fc2(GELU(fc1(LN2(x))))
* ``Block("llama", ...)`` pre-norm LLaMA block (causal attention, no biases):
      x = x + o(attn(q(n1), k(n1), v(n1))),    n1 = RMSNorm1(x)
      x = x + down(SiLU(gate(n2)) * up(n2)),   n2 = RMSNorm2(x)

Attention is context, not the method: torch SDPA (whatever fused backend it
picks), identical in the exact and our block, so its saved tensors cancel in
every comparison; rotary embeddings are left out (they save no activations).

Fine-tuning regimes (``tuning``) fix which linears keep their input for
backward (a frozen linear's input gradient needs only its weight):

    full         every linear trainable (Full-Tuning)
    lora_qv      LoRA on q and v, everything else frozen
    lora_all     LoRA on every linear (QLoRA's choice)
    lora_fa_qv   LoRA-FA on q and v: A frozen, only A z saved
    lora_fa_all  LoRA-FA on every linear
    frozen_ffn   attention linears trainable, FFN frozen

LoRA (Eq. 4): z' = W z + B A z + b with A [r, p], B [p', r].

``exact`` (the constructor's block) is the reference composition the paper
compares against: LayerNorm / RMSNorm with affine (fp32 as under AMP when
``norm_fp32``; a single-kernel norm that saves its input and
per-row statistics), exact GELU / SiLU, unmerged linears.  ``to_ours()``
returns the same function with the method applied: the norm affine merged into
every consumer linear (W~ = W diag(alpha), b~ = W beta + b; for a
LoRA consumer A~ = A diag(alpha) and the constant A beta kept as the LoRA-A
bias, so the merged block computes exactly the same function at the current
parameters), MS-LN / MS-RMSNorm, ReGELU2 / fused ReSwiGLU2.  MS norms share
their saved y with the consumer linears only where Prop. 5.1 condition 3
holds: where every consumer is frozen or LoRA-FA
the MS norm's y is kept for nobody else and the norm saves as much as the
plain norm of the same dtype (its input replaced by its output).
"""
from __future__ import annotations

import copy

import torch
import torch.nn.functional as F

from . import modules

TUNINGS = ("full", "lora_qv", "lora_all", "lora_fa_qv", "lora_fa_all", "frozen_ffn")
LINEAR_MODES = ("full", "frozen", "lora", "lora_fa")


def linear_modes(arch: str, tuning: str) -> dict:
    """Mode of every linear of the block under a fine-tuning regime."""
    attn = ["q", "k", "v", "proj" if arch == "vit" else "o"]
    ffn = ["fc1", "fc2"] if arch == "vit" else ["gate", "up", "down"]
    if tuning not in TUNINGS:
        raise ValueError(f"tuning must be one of {TUNINGS}")
    m = {}
    for n in attn + ffn:
        if tuning == "full":
            m[n] = "full"
        elif tuning == "lora_all":
            m[n] = "lora"
        elif tuning == "lora_fa_all":
            m[n] = "lora_fa"
        elif tuning in ("lora_qv", "lora_fa_qv"):
            m[n] = ("lora" if tuning == "lora_qv" else "lora_fa") if n in ("q", "v") else "frozen"
        else:  # frozen_ffn
            m[n] = "full" if n in attn else "frozen"
    return m


def saves_input(mode: str) -> bool:
    """Does a linear in this mode keep its full input for backward? (full:
    for dW; LoRA: for dA.  Frozen and LoRA-FA do not.)"""
    return mode in ("full", "lora")


class Linear(torch.nn.Module):
    """y = W x + b (+ scale * B (A x + a_bias)): a pretrained linear with an
    optional LoRA / LoRA-FA adapter; requires_grad follows the mode."""

    def __init__(self, cin, cout, bias=True, mode="full", rank=4, dtype=torch.bfloat16, device="cuda",
                 gen=None, lora_init_b=0.0):
        super().__init__()
        if mode not in LINEAR_MODES:
            raise ValueError(f"mode must be one of {LINEAR_MODES}")
        self.in_features, self.out_features, self.mode, self.rank = cin, cout, mode, rank
        w = torch.randn(cout, cin, generator=gen) / cin ** 0.5
        self.weight = torch.nn.Parameter(w.to(device=device, dtype=dtype))
        self.bias = (torch.nn.Parameter((0.02 * torch.randn(cout, generator=gen)).to(device=device, dtype=dtype))
                     if bias else None)
        self.lora_A = self.lora_B = self.lora_a_bias = None
        self.scale = 1.0
        if mode in ("lora", "lora_fa"):
            a = torch.randn(rank, cin, generator=gen) / cin ** 0.5
            b = lora_init_b * torch.randn(cout, rank, generator=gen)     # LoRA initialises B = 0
            self.lora_A = torch.nn.Parameter(a.to(device=device, dtype=dtype))
            self.lora_B = torch.nn.Parameter(b.to(device=device, dtype=dtype))
        self._apply_mode()

    def _apply_mode(self):
        full = self.mode == "full"
        self.weight.requires_grad_(full)
        if self.bias is not None:
            self.bias.requires_grad_(full)
        if self.lora_A is not None:
            self.lora_A.requires_grad_(self.mode == "lora")
            self.lora_B.requires_grad_(True)
        if self.lora_a_bias is not None:
            self.lora_a_bias.requires_grad_(False)

    def forward(self, x):
        y = F.linear(x, self.weight, self.bias)
        if self.lora_A is not None:
            y = y + self.scale * F.linear(F.linear(x, self.lora_A, self.lora_a_bias), self.lora_B)
        return y


@torch.no_grad()
def fold_affine(linears, alpha, beta):
    """Merge a norm's affine (alpha, beta) into every consumer linear
    (P:L509-517): W~ = W diag(alpha), b~ = W beta + b; a LoRA adapter's A
    becomes A diag(alpha) with the constant A beta as its bias, so
    B A (alpha * zh + beta) = B (A~ zh + A beta) exactly."""
    from .merge import merge_ln
    for lin in linears:
        w, b = merge_ln(lin.weight, lin.bias, alpha, beta)
        lin.weight.copy_(w)
        if b is not None:
            if lin.bias is None:
                lin.bias = torch.nn.Parameter(b)
            else:
                lin.bias.copy_(b)
        if lin.lora_A is not None:
            a, ab = merge_ln(lin.lora_A, None, alpha, beta)
            lin.lora_A.copy_(a)
            if ab is not None:
                lin.lora_a_bias = torch.nn.Parameter(ab)
        lin._apply_mode()


class _NormRefFn(torch.autograd.Function):
    """Reference LayerNorm / RMSNorm with affine as ONE kernel would run it
    (the Fig. 5/6 assumption): saves its input (in the norm's
    compute dtype), per-row statistics and the affine parameters."""

    @staticmethod
    def forward(ctx, x, alpha, beta, eps, ln, fp32, out_dtype=None):
        xc = x.float() if fp32 else x
        xf = xc.float()
        mu = xf.mean(-1, keepdim=True) if ln else torch.zeros_like(xf[..., :1])
        rstd = torch.rsqrt(((xf - mu) ** 2).mean(-1, keepdim=True) + eps)
        zh = (xf - mu) * rstd
        z = zh * alpha.float() + (beta.float() if beta is not None else 0.0)
        if ln:
            ctx.save_for_backward(xc, mu.squeeze(-1), rstd.squeeze(-1), alpha, beta)
        else:
            ctx.save_for_backward(xc, rstd.squeeze(-1), alpha)
        ctx.ln = ln
        ctx.in_dtype = x.dtype
        return z.to(out_dtype or x.dtype)

    @staticmethod
    def backward(ctx, gz):
        if ctx.ln:
            xc, mu, rstd, alpha, beta = ctx.saved_tensors
        else:
            (xc, rstd, alpha), mu = ctx.saved_tensors, None
        xf = xc.float()
        r = rstd.unsqueeze(-1)
        zh = (xf - mu.unsqueeze(-1)) * r if ctx.ln else xf * r
        g = gz.float()
        ga = g * alpha.float()
        dx = r * (ga - (ga.mean(-1, keepdim=True) if ctx.ln else 0.0) - zh * (ga * zh).mean(-1, keepdim=True))
        flat = lambda t: t.reshape(-1, t.shape[-1])
        dalpha = (flat(g) * flat(zh)).sum(0).to(alpha.dtype) if alpha.requires_grad else None
        dbeta = None
        if ctx.ln and beta is not None and beta.requires_grad:
            dbeta = flat(g).sum(0).to(beta.dtype)
        return dx.to(ctx.in_dtype), dalpha, dbeta, None, None, None, None


class NormRef(torch.nn.Module):
    def __init__(self, p, ln: bool, eps=1e-6, fp32=True, device="cuda", gen=None, trainable=False, out_dtype=None):
        super().__init__()
        self.ln, self.eps, self.fp32, self.p, self.out_dtype = ln, eps, fp32, p, out_dtype
        self.weight = torch.nn.Parameter((1 + 0.1 * torch.randn(p, generator=gen)).to(device),
                                         requires_grad=trainable)
        self.bias = (torch.nn.Parameter((0.1 * torch.randn(p, generator=gen)).to(device), requires_grad=trainable)
                     if ln else None)

    def forward(self, x):
        return _NormRefFn.apply(x, self.weight, self.bias, self.eps, self.ln, self.fp32, self.out_dtype)


class Attention(torch.nn.Module):
    """Multi-head SDPA over [b, n, c] projections (context, not the method)."""

    def __init__(self, heads: int, causal: bool):
        super().__init__()
        self.heads, self.causal = heads, causal

    def forward(self, q, k, v):
        b, n, c = q.shape
        sh = lambda t: t.view(b, n, self.heads, c // self.heads).transpose(1, 2)
        o = F.scaled_dot_product_attention(sh(q), sh(k), sh(v), is_causal=self.causal)
        return o.transpose(1, 2).reshape(b, n, c)


class SwiGLURef(torch.nn.Module):
    def forward(self, gate, up):
        return F.silu(gate) * up


class Block(torch.nn.Module):
    def __init__(self, arch: str, c: int, hidden: int, heads: int, tuning: str = "full", rank: int = 4,
                 eps: float = 1e-6, dtype=torch.bfloat16, device="cuda", seed: int = 0, norm_fp32: bool = True,
                 lora_init_b: float = 0.0, residual_fp32: bool = False):
        super().__init__()
        if arch not in ("vit", "llama"):
            raise ValueError("arch must be 'vit' or 'llama'")
        g = torch.Generator(device="cpu").manual_seed(seed)
        self.arch, self.c, self.hidden, self.tuning, self.eps = arch, c, hidden, tuning, eps
        # residual_fp32: the AMP layout -- fp32 residual stream, 16-bit linears; the
        # norms read fp32 and emit the linears' dtype (ours: msln/msrms_*_mixed)
        self.residual_fp32, self.dtype = residual_fp32, dtype
        nout = dtype if residual_fp32 else None
        ln, bias = arch == "vit", arch == "vit"
        self.modes = linear_modes(arch, tuning)
        mk = lambda name, i, o: Linear(i, o, bias, self.modes[name], rank, dtype, device, g, lora_init_b)
        self.norm1 = NormRef(c, ln, eps, norm_fp32, device, g, out_dtype=nout)
        self.q, self.k, self.v = mk("q", c, c), mk("k", c, c), mk("v", c, c)
        self.attn = Attention(heads, causal=arch == "llama")
        self.norm2 = NormRef(c, ln, eps, norm_fp32, device, g, out_dtype=nout)
        if arch == "vit":
            self.proj = mk("proj", c, c)
            self.fc1, self.fc2 = mk("fc1", c, hidden), mk("fc2", hidden, c)
            self.act = torch.nn.GELU()
        else:
            self.o = mk("o", c, c)
            self.gate, self.up, self.down = mk("gate", c, hidden), mk("up", c, hidden), mk("down", hidden, c)
            self.act = SwiGLURef()
        self.ms_norm = self.approx_act = False

    # Prop. 5.1 condition 3: some consumer of the norm keeps its input
    def norm_shared(self, which: int) -> bool:
        cons = ["q", "k", "v"] if which == 1 else (["fc1"] if self.arch == "vit" else ["gate", "up"])
        return any(saves_input(self.modes[n]) for n in cons)

    def to_ours(self, norm: bool = True, act: bool = True):
        """The same block with the method applied (norm: merge + MS norms;
        act: ReGELU2 / fused ReSwiGLU2)."""
        m = copy.deepcopy(self)
        if norm:
            cons2 = [m.fc1] if m.arch == "vit" else [m.gate, m.up]
            for nm, cons in ((m.norm1, [m.q, m.k, m.v]), (m.norm2, cons2)):
                fold_affine(cons, nm.weight.detach(), None if nm.bias is None else nm.bias.detach())
            ms = modules.MSLayerNorm if m.arch == "vit" else modules.MSRMSNorm
            od = m.dtype if m.residual_fp32 else None
            m.norm1, m.norm2 = ms(m.c, m.eps, out_dtype=od), ms(m.c, m.eps, out_dtype=od)
            m.ms_norm = True
        if act:
            m.act = modules.ReGELU2() if m.arch == "vit" else modules.ReSwiGLU2()
            m.approx_act = True
        return m

    def forward(self, x):
        n1 = self.norm1(x)
        a = self.attn(self.q(n1), self.k(n1), self.v(n1))
        x = x + (self.proj(a) if self.arch == "vit" else self.o(a))
        n2 = self.norm2(x)
        if self.arch == "vit":
            h = self.fc2(self.act(self.fc1(n2)))
        else:
            h = self.down(self.act(self.gate(n2), self.up(n2)))
        return x + h


# Decoded Fig. 5 / Fig. 6 unit model (unit = one [b, n, c]
# 16-bit tensor; norms in fp32): full tuning, exact and ours.
def unit_model(arch: str, expansion: float) -> dict:
    if arch == "vit":   # LN 2+2, qkv in 1, q/k/v 3, attn out 1, proj in 1, fc1 in 1, GELU in 4, fc2 in 4
        exact = 2 + 1 + 3 + 1 + 1 + 2 + 1 + 2 * expansion
        ours = 1 + 3 + 1 + 1 + 1 + expansion / 8 + expansion
    else:               # RMS 2+2, qkv in 1, q/k/v 3, attn out 1, o in 1, gate/up in 1, SiLU in, silu, up, down in
        exact = 2 + 1 + 3 + 1 + 1 + 2 + 1 + 4 * expansion
        ours = 1 + 3 + 1 + 1 + 1 + 2 * expansion + expansion / 8 + expansion
    return {"exact_units": exact, "ours_units": ours, "saved_fraction": 1 - ours / exact}


def activation_bytes(block: torch.nn.Module, x: torch.Tensor, by_module: bool = False):
    """Activation bytes `block(x)` keeps for backward, deduplicated by
    storage, excluding parameters (weights are not activations).  With
    by_module, also {module name: bytes} attributing each storage to the
    innermost module whose forward first saved it."""
    params = {p.untyped_storage().data_ptr() for p in block.parameters()}
    seen, owner, stack = {}, {}, [""]
    hooks = []
    if by_module:
        for name, mod in block.named_modules():
            if name:
                def pre(m, a, n=name):
                    stack.append(n)

                def post(m, a, o):
                    stack.pop()
                hooks.append(mod.register_forward_pre_hook(pre))
                hooks.append(mod.register_forward_hook(post))

    def pack(t):
        st = t.untyped_storage()
        key = st.data_ptr()
        if key not in params and key not in seen:
            seen[key] = st.nbytes()
            owner[key] = stack[-1]
        return t

    try:
        with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
            out = block(x)
        del out
    finally:
        for h in hooks:
            h.remove()
    total = int(sum(seen.values()))
    if not by_module:
        return total
    per = {}
    for k, v in seen.items():
        per[owner[k]] = per.get(owner[k], 0) + v
    return total, per
