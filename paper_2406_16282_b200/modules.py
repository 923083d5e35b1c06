"""Autograd functions and modules over the C ABI.

* ReGELU2 / ReSiLU2 save only the packed 2-bit codes.
* MSLayerNorm / MSRMSNorm are affine-free (the affine is merged into the next
  linear layer) and save (y, rstd): y is the tensor the next
  linear layer saves anyway, so it is stored once (Prop. 5.1).

``saved_bytes`` measures the activation memory a forward retains for
backward (the "activation bytes saved per layer" half of the metric, a7),
deduplicating tensors that share storage.
"""
from __future__ import annotations

import torch

from . import ops


class ReGELU2Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        y, codes = ops.regelu2_fwd(x.contiguous())
        ctx.save_for_backward(codes)
        return y

    @staticmethod
    def backward(ctx, dy):
        (codes,) = ctx.saved_tensors
        return ops.regelu2_bwd(dy.contiguous(), codes)


class ReSiLU2Fn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x):
        y, codes = ops.resilu2_fwd(x.contiguous())
        ctx.save_for_backward(codes)
        return y

    @staticmethod
    def backward(ctx, dy):
        (codes,) = ctx.saved_tensors
        return ops.resilu2_bwd(dy.contiguous(), codes)


class MSLayerNormFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, eps):
        y, rstd = ops.msln_fwd(x.contiguous(), eps)
        ctx.save_for_backward(y, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        y, rstd = ctx.saved_tensors
        return ops.msln_bwd(dy.contiguous(), y, rstd), None


class MSRMSNormFn(torch.autograd.Function):
    @staticmethod
    def forward(ctx, x, eps):
        y, rstd = ops.msrms_fwd(x.contiguous(), eps)
        ctx.save_for_backward(y, rstd)
        return y

    @staticmethod
    def backward(ctx, dy):
        y, rstd = ctx.saved_tensors
        return ops.msrms_bwd(dy.contiguous(), y, rstd), None


class MSNormMixedFn(torch.autograd.Function):
    """fp32 residual x -> 16-bit y (the next linear's input dtype); saves
    (y, rstd); backward returns the fp32 dx of the residual stream."""

    @staticmethod
    def forward(ctx, x, eps, out_dtype, ln):
        fwd = ops.msln_fwd_mixed if ln else ops.msrms_fwd_mixed
        y, rstd = fwd(x.contiguous(), eps, out_dtype)
        ctx.save_for_backward(y, rstd)
        ctx.ln = ln
        return y

    @staticmethod
    def backward(ctx, dy):
        y, rstd = ctx.saved_tensors
        bwd = ops.msln_bwd_mixed if ctx.ln else ops.msrms_bwd_mixed
        return bwd(dy.to(y.dtype).contiguous(), y, rstd), None, None, None


class ReSwiGLU2Fn(torch.autograd.Function):
    """h = SiLU(gate) * up with ReSiLU2's backward, fused; saves (up, a, codes)
    where a = SiLU(gate) -- 2b + 1/4 bytes per element instead of 3b."""

    @staticmethod
    def forward(ctx, gate, up):
        h, a, codes = ops.reswiglu2_fwd(gate.contiguous(), up.contiguous())
        ctx.save_for_backward(up, a, codes)
        return h

    @staticmethod
    def backward(ctx, dh):
        up, a, codes = ctx.saved_tensors
        dgate, dup = ops.reswiglu2_bwd(dh.contiguous(), up.contiguous(), a, codes)
        return dgate, dup


class ReSwiGLU2(torch.nn.Module):
    def forward(self, gate, up):
        return ReSwiGLU2Fn.apply(gate, up)


class ReGELU2(torch.nn.Module):
    def forward(self, x):
        return ReGELU2Fn.apply(x)


class ReSiLU2(torch.nn.Module):
    def forward(self, x):
        return ReSiLU2Fn.apply(x)


class MSLayerNorm(torch.nn.Module):
    """Affine-free LayerNorm whose backward needs only (y, rstd).  With
    ``out_dtype`` (bfloat16 / float16) an fp32 input is normalised straight
    into that dtype (msln_fwd_mixed: AMP's fp32 norm feeding a 16-bit linear)."""

    def __init__(self, normalized_shape: int, eps: float = 1e-6, out_dtype=None):
        super().__init__()
        self.normalized_shape = int(normalized_shape)
        self.eps = float(eps)
        self.out_dtype = out_dtype

    def forward(self, x):
        if x.shape[-1] != self.normalized_shape:
            raise ValueError("last dimension mismatch")
        if self.out_dtype is not None and x.dtype == torch.float32 and self.out_dtype != torch.float32:
            return MSNormMixedFn.apply(x, self.eps, self.out_dtype, True)
        return MSLayerNormFn.apply(x, self.eps)


class MSRMSNorm(torch.nn.Module):
    def __init__(self, normalized_shape: int, eps: float = 1e-6, out_dtype=None):
        super().__init__()
        self.normalized_shape = int(normalized_shape)
        self.eps = float(eps)
        self.out_dtype = out_dtype

    def forward(self, x):
        if x.shape[-1] != self.normalized_shape:
            raise ValueError("last dimension mismatch")
        if self.out_dtype is not None and x.dtype == torch.float32 and self.out_dtype != torch.float32:
            return MSNormMixedFn.apply(x, self.eps, self.out_dtype, False)
        return MSRMSNormFn.apply(x, self.eps)


def saved_bytes(fn, *inputs) -> int:
    """Bytes of activation state ``fn(*inputs)`` saves for backward, with
    tensors that share storage counted once (storage data_ptr)."""
    seen = {}

    def pack(t):
        st = t.untyped_storage()
        seen[(st.data_ptr(), t.device)] = st.nbytes()
        return t

    with torch.autograd.graph.saved_tensors_hooks(pack, lambda t: t):
        out = fn(*inputs)
    del out
    return int(sum(seen.values()))
