"""Thin Python binding over the C ABI: same names as include/lmbp.h.

Argument marshalling only -- every step runs in liblmbp.so's CUDA kernels.
PyTorch supplies device memory and the current stream.  Tensors must be CUDA,
contiguous, and fp32 / bf16 / fp16; outputs are allocated when not given.
Activations treat the tensor as one flat sequence (rows = numel / last dim,
cols = last dim); norms normalise over the last dimension.
"""
from __future__ import annotations

import torch

from . import _lib
from ._lib import check, lib

_DT = {torch.float32: _lib.LMBP_F32, torch.bfloat16: _lib.LMBP_BF16, torch.float16: _lib.LMBP_F16}


def codes_bytes(n: int) -> int:
    return int(lib().lmbp_codes_bytes(int(n)))


def _dtype(t: torch.Tensor) -> int:
    try:
        return _DT[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported dtype {t.dtype}; expected float32, bfloat16 or float16") from None


def _rc(t: torch.Tensor):
    if t.dim() == 0:
        return 1, 1
    cols = t.shape[-1]
    return (t.numel() // cols if cols else 0), cols


def _need(t: torch.Tensor, name: str) -> torch.Tensor:
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (no CPU fallback)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")
    return t


def _stream(stream, dev: torch.device) -> int:
    if stream is None:
        stream = torch.cuda.current_stream(dev)
    elif isinstance(stream, torch.cuda.Stream):
        if stream.device != dev:
            raise ValueError(f"stream is on {stream.device}, tensors on {dev}")
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _device(fn: str, *ts: torch.Tensor) -> torch.device:
    """The one device all tensors of a call live on (the library launches on
    the current device, so a call is made with that device current)."""
    dev = ts[0].device
    for t in ts[1:]:
        if t.device != dev:
            raise ValueError(f"{fn}: tensors on different devices ({dev}, {t.device})")
    return dev


_ENTRY = {}


def _entry(fn: str):
    f = _ENTRY.get(fn)
    if f is None:
        f = _ENTRY[fn] = getattr(lib(), fn)
    return f


def _launch(fn: str, dev: torch.device, stream, *args) -> None:
    """Call entry point fn(*args, stream) with dev current; raise on a status.
    (The device switch is skipped when dev already is the current device: it
    is most of the host cost of a call.)"""
    s = _stream(stream, dev)
    if dev.index is None or dev.index == torch.cuda.current_device():
        status = _entry(fn)(*args, s)
    else:
        with torch.cuda.device(dev):
            status = _entry(fn)(*args, s)
    if status:
        check(fn, status)


def _act_fwd(fn: str, x, y, codes, stream):
    _need(x, "x")
    y = torch.empty_like(x) if y is None else _need(y, "y")
    n = x.numel()
    nc = codes_bytes(n)
    codes = torch.empty(nc, dtype=torch.uint8, device=x.device) if codes is None else _need(codes, "codes")
    if y.shape != x.shape or y.dtype != x.dtype or codes.numel() != nc:
        raise ValueError(f"{fn}: shape/dtype mismatch")
    rows, cols = _rc(x)
    if n == 0:
        return y, codes
    _launch(fn, _device(fn, x, y, codes), stream, x.data_ptr(), y.data_ptr(), codes.data_ptr(), rows, cols,
            _dtype(x))
    return y, codes


def _act_bwd(fn: str, dy, codes, dx, stream):
    _need(dy, "dy")
    _need(codes, "codes")
    dx = torch.empty_like(dy) if dx is None else _need(dx, "dx")
    n = dy.numel()
    nc = codes_bytes(n)
    if codes.numel() != nc or codes.dtype != torch.uint8:
        raise ValueError(f"{fn}: codes must be uint8[{nc}] (S:L174)")
    if dx.shape != dy.shape or dx.dtype != dy.dtype:
        raise ValueError(f"{fn}: shape/dtype mismatch")
    rows, cols = _rc(dy)
    if n == 0:
        return dx
    _launch(fn, _device(fn, dy, codes, dx), stream, dy.data_ptr(), codes.data_ptr(), dx.data_ptr(), rows, cols,
            _dtype(dy))
    return dx


def regelu2_fwd(x, y=None, codes=None, stream=None):
    """ReGELU2 forward: (y = GELU(x), packed 2-bit codes).  lmbp.h regelu2_fwd."""
    return _act_fwd("regelu2_fwd", x, y, codes, stream)


def regelu2_bwd(dy, codes, dx=None, stream=None):
    """ReGELU2 backward: dx = dy * s[code].  lmbp.h regelu2_bwd."""
    return _act_bwd("regelu2_bwd", dy, codes, dx, stream)


def resilu2_fwd(x, y=None, codes=None, stream=None):
    """ReSiLU2 forward: (y = SiLU(x), packed 2-bit codes).  lmbp.h resilu2_fwd."""
    return _act_fwd("resilu2_fwd", x, y, codes, stream)


def resilu2_bwd(dy, codes, dx=None, stream=None):
    """ReSiLU2 backward.  lmbp.h resilu2_bwd."""
    return _act_bwd("resilu2_bwd", dy, codes, dx, stream)


def _norm_fwd(fn, x, eps, y, rstd, stream):
    _need(x, "x")
    rows, cols = _rc(x)
    y = torch.empty_like(x) if y is None else _need(y, "y")
    rstd = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device) if rstd is None else _need(rstd, "rstd")
    if y.shape != x.shape or y.dtype != x.dtype or rstd.numel() != rows or rstd.dtype != torch.float32:
        raise ValueError(f"{fn}: shape/dtype mismatch")
    _launch(fn, _device(fn, x, y, rstd), stream, x.data_ptr(), y.data_ptr(), rstd.data_ptr(), rows, cols,
            float(eps), _dtype(x))
    return y, rstd


def _norm_bwd(fn, dy, y, rstd, dx, stream):
    _need(dy, "dy")
    _need(y, "y")
    _need(rstd, "rstd")
    rows, cols = _rc(dy)
    dx = torch.empty_like(dy) if dx is None else _need(dx, "dx")
    if y.shape != dy.shape or y.dtype != dy.dtype or rstd.numel() != rows or dx.shape != dy.shape \
            or rstd.dtype != torch.float32 or dx.dtype != dy.dtype:
        raise ValueError(f"{fn}: token/shape mismatch (S:L266)")
    _launch(fn, _device(fn, dy, y, rstd, dx), stream, dy.data_ptr(), y.data_ptr(), rstd.data_ptr(), dx.data_ptr(),
            rows, cols, _dtype(dy))
    return dx


def msln_fwd(x, eps=1e-6, y=None, rstd=None, stream=None):
    """MS-LN forward (Alg. 2): (y, rstd).  lmbp.h msln_fwd."""
    return _norm_fwd("msln_fwd", x, eps, y, rstd, stream)


def msln_bwd(dy, y, rstd, dx=None, stream=None):
    """MS-LN backward from (dy, y, rstd) only.  lmbp.h msln_bwd."""
    return _norm_bwd("msln_bwd", dy, y, rstd, dx, stream)


def msrms_fwd(x, eps=1e-6, y=None, rstd=None, stream=None):
    """MS-RMSNorm forward (Alg. 3).  lmbp.h msrms_fwd."""
    return _norm_fwd("msrms_fwd", x, eps, y, rstd, stream)


def msrms_bwd(dy, y, rstd, dx=None, stream=None):
    """MS-RMSNorm backward.  lmbp.h msrms_bwd."""
    return _norm_bwd("msrms_bwd", dy, y, rstd, dx, stream)


def _norm_fwd_mixed(fn, x, eps, out_dtype, y, rstd, stream):
    _need(x, "x")
    if x.dtype != torch.float32:
        raise ValueError(f"{fn}: x must be float32 (the fp32 residual stream)")
    if out_dtype not in (torch.bfloat16, torch.float16):
        raise ValueError(f"{fn}: out_dtype must be bfloat16 or float16")
    rows, cols = _rc(x)
    y = torch.empty(x.shape, dtype=out_dtype, device=x.device) if y is None else _need(y, "y")
    rstd = torch.empty(x.shape[:-1], dtype=torch.float32, device=x.device) if rstd is None else _need(rstd, "rstd")
    if y.shape != x.shape or y.dtype != out_dtype or rstd.numel() != rows or rstd.dtype != torch.float32:
        raise ValueError(f"{fn}: shape/dtype mismatch")
    _launch(fn, _device(fn, x, y, rstd), stream, x.data_ptr(), y.data_ptr(), rstd.data_ptr(), rows, cols,
            float(eps), _dtype(y))
    return y, rstd


def _norm_bwd_mixed(fn, dy, y, rstd, dx, stream):
    for t, nm in ((dy, "dy"), (y, "y"), (rstd, "rstd")):
        _need(t, nm)
    if dy.dtype not in (torch.bfloat16, torch.float16) or y.dtype != dy.dtype:
        raise ValueError(f"{fn}: dy and y must share a 16-bit dtype")
    rows, cols = _rc(dy)
    dx = torch.empty(dy.shape, dtype=torch.float32, device=dy.device) if dx is None else _need(dx, "dx")
    if y.shape != dy.shape or rstd.numel() != rows or rstd.dtype != torch.float32 or dx.shape != dy.shape \
            or dx.dtype != torch.float32:
        raise ValueError(f"{fn}: token/shape mismatch (S:L266)")
    _launch(fn, _device(fn, dy, y, rstd, dx), stream, dy.data_ptr(), y.data_ptr(), rstd.data_ptr(), dx.data_ptr(),
            rows, cols, _dtype(dy))
    return dx


def msln_fwd_mixed(x, eps=1e-6, out_dtype=torch.bfloat16, y=None, rstd=None, stream=None):
    """MS-LN forward from an fp32 residual stream to a 16-bit y (AMP).  lmbp.h msln_fwd_mixed."""
    return _norm_fwd_mixed("msln_fwd_mixed", x, eps, out_dtype, y, rstd, stream)


def msln_bwd_mixed(dy, y, rstd, dx=None, stream=None):
    """MS-LN backward: 16-bit (dy, y) + rstd -> fp32 dx.  lmbp.h msln_bwd_mixed."""
    return _norm_bwd_mixed("msln_bwd_mixed", dy, y, rstd, dx, stream)


def msrms_fwd_mixed(x, eps=1e-6, out_dtype=torch.bfloat16, y=None, rstd=None, stream=None):
    """MS-RMSNorm forward, fp32 x -> 16-bit y.  lmbp.h msrms_fwd_mixed."""
    return _norm_fwd_mixed("msrms_fwd_mixed", x, eps, out_dtype, y, rstd, stream)


def msrms_bwd_mixed(dy, y, rstd, dx=None, stream=None):
    """MS-RMSNorm backward, 16-bit (dy, y) -> fp32 dx.  lmbp.h msrms_bwd_mixed."""
    return _norm_bwd_mixed("msrms_bwd_mixed", dy, y, rstd, dx, stream)


def step_table(kind: str):
    """The kernels' binary32 (thresholds[3], levels[4]) for 'gelu' / 'silu'."""
    import ctypes
    t = (ctypes.c_float * 3)()
    lv = (ctypes.c_float * 4)()
    check("lmbp_step_table", lib().lmbp_step_table({"gelu": _lib.LMBP_GELU, "silu": _lib.LMBP_SILU}[kind],
                                                   ctypes.addressof(t), ctypes.addressof(lv)))
    return list(t), list(lv)


def reswiglu2_fwd(gate, up, h=None, a=None, codes=None, stream=None):
    """Fused ReSwiGLU2 forward: (h = RN(a * up), a = RN(SiLU(gate)), codes of
    gate).  lmbp.h reswiglu2_fwd."""
    _need(gate, "gate")
    _need(up, "up")
    n = gate.numel()
    h = torch.empty_like(gate) if h is None else _need(h, "h")
    a = torch.empty_like(gate) if a is None else _need(a, "a")
    codes = (torch.empty(codes_bytes(n), dtype=torch.uint8, device=gate.device) if codes is None
             else _need(codes, "codes"))
    for t in (up, h, a):
        if t.shape != gate.shape or t.dtype != gate.dtype:
            raise ValueError("reswiglu2_fwd: shape/dtype mismatch")
    if codes.numel() != codes_bytes(n):
        raise ValueError("reswiglu2_fwd: codes size")
    rows, cols = _rc(gate)
    if n == 0:
        return h, a, codes
    _launch("reswiglu2_fwd", _device("reswiglu2_fwd", gate, up, h, a, codes), stream, gate.data_ptr(),
            up.data_ptr(), h.data_ptr(), a.data_ptr(), codes.data_ptr(), rows, cols, _dtype(gate))
    return h, a, codes


def reswiglu2_bwd(dh, up, a, codes, dgate=None, dup=None, stream=None):
    """Fused ReSwiGLU2 backward: (dgate, dup).  lmbp.h reswiglu2_bwd."""
    for t, nm in ((dh, "dh"), (up, "up"), (a, "a"), (codes, "codes")):
        _need(t, nm)
    n = dh.numel()
    dgate = torch.empty_like(dh) if dgate is None else _need(dgate, "dgate")
    dup = torch.empty_like(dh) if dup is None else _need(dup, "dup")
    for t in (up, a, dgate, dup):
        if t.shape != dh.shape or t.dtype != dh.dtype:
            raise ValueError("reswiglu2_bwd: shape/dtype mismatch")
    if codes.numel() != codes_bytes(n) or codes.dtype != torch.uint8:
        raise ValueError("reswiglu2_bwd: codes size")
    rows, cols = _rc(dh)
    if n == 0:
        return dgate, dup
    _launch("reswiglu2_bwd", _device("reswiglu2_bwd", dh, up, a, codes, dgate, dup), stream, dh.data_ptr(),
            up.data_ptr(), a.data_ptr(), codes.data_ptr(), dgate.data_ptr(), dup.data_ptr(), rows, cols, _dtype(dh))
    return dgate, dup


# ---------------------------------------------------------------------------
# k-bit step activations (lmbp.h stepact_*)
# ---------------------------------------------------------------------------
def codes_bytes_k(n: int, k: int) -> int:
    return int(lib().lmbp_codes_bytes_k(int(n), int(k)))


def _dbl(vals):
    import ctypes
    arr = (ctypes.c_double * len(vals))(*[float(v) for v in vals])
    return arr, ctypes.addressof(arr)


def _check_table(fn: str, k: int, vals, want: int, what: str):
    """The C ABI reads exactly `want` doubles: refuse any other length here,
    before a short host array could be read past its end."""
    if int(k) not in (1, 2, 3, 4):
        raise ValueError(f"{fn}: k must be 1, 2, 3 or 4 (got {k})")
    if len(vals) != want:
        raise ValueError(f"{fn}: {what} needs exactly {want} entries for k = {k} (got {len(vals)})")


def stepact_fwd(x, act: str, k: int, thresholds, y=None, codes=None, stream=None):
    """Forward of a k-bit step activation: (y = act(x), k-bit codes)."""
    _check_table("stepact_fwd", k, thresholds, (1 << int(k)) - 1, "thresholds")
    _need(x, "x")
    n = x.numel()
    y = torch.empty_like(x) if y is None else _need(y, "y")
    codes = (torch.empty(codes_bytes_k(n, k), dtype=torch.uint8, device=x.device) if codes is None
             else _need(codes, "codes"))
    if y.shape != x.shape or y.dtype != x.dtype or codes.numel() != codes_bytes_k(n, k):
        raise ValueError("stepact_fwd: shape/dtype/codes mismatch")
    rows, cols = _rc(x)
    keep, ptr = _dbl(thresholds)
    if n == 0:
        return y, codes
    _launch("stepact_fwd", _device("stepact_fwd", x, y, codes), stream,
            {"gelu": _lib.LMBP_GELU, "silu": _lib.LMBP_SILU}[act], int(k), ptr, x.data_ptr(), y.data_ptr(),
            codes.data_ptr(), rows, cols, _dtype(x))
    return y, codes


def stepact_bwd(dy, codes, k: int, levels, dx=None, stream=None):
    """Backward of a k-bit step activation: dx = dy * levels[code]."""
    _check_table("stepact_bwd", k, levels, 1 << int(k), "levels")
    _need(dy, "dy")
    _need(codes, "codes")
    if codes.dtype != torch.uint8:
        raise ValueError("stepact_bwd: codes must be uint8")
    n = dy.numel()
    dx = torch.empty_like(dy) if dx is None else _need(dx, "dx")
    if codes.numel() != codes_bytes_k(n, k) or dx.shape != dy.shape or dx.dtype != dy.dtype:
        raise ValueError("stepact_bwd: shape/codes mismatch")
    rows, cols = _rc(dy)
    keep, ptr = _dbl(levels)
    if n == 0:
        return dx
    _launch("stepact_bwd", _device("stepact_bwd", dy, codes, dx), stream, int(k), ptr, dy.data_ptr(),
            codes.data_ptr(), dx.data_ptr(), rows, cols, _dtype(dy))
    return dx


# ---------------------------------------------------------------------------
# Offline coefficient fitter (lmbp.h lmbp_fit_*)
# ---------------------------------------------------------------------------
_ACT = {"gelu": _lib.LMBP_GELU, "silu": _lib.LMBP_SILU}
_OBJ = {"h": _lib.LMBP_FIT_H, "dh": _lib.LMBP_FIT_DH}


def fit_n_params(k: int) -> int:
    """2 m - 1 parameters (m - 1 weights, m thresholds), m = 2^k - 1."""
    return 2 * ((1 << int(k)) - 1) - 1


def fit_bounds(act: str, eps: float = 1e-8):
    """[A, B] of App. E for tail tolerance eps (host only)."""
    import ctypes
    A, B = ctypes.c_double(), ctypes.c_double()
    check("lmbp_fit_bounds", lib().lmbp_fit_bounds(_ACT[act], float(eps), ctypes.byref(A), ctypes.byref(B)))
    return A.value, B.value


def fit_objective(theta, act: str, k: int = 2, objective: str = "h", eps: float = 1e-8, J=None, stream=None):
    """J(theta) for every row of a CUDA float64 tensor theta [n, P]."""
    _need(theta, "theta")
    P = fit_n_params(k)
    if theta.dtype != torch.float64 or theta.dim() != 2 or theta.shape[1] != P:
        raise ValueError(f"theta must be float64 [n, {P}]")
    n = theta.shape[0]
    J = torch.empty(n, dtype=torch.float64, device=theta.device) if J is None else _need(J, "J")
    if J.dtype != torch.float64 or J.numel() != n:
        raise ValueError("J must be float64 [n]")
    _launch("lmbp_fit_objective", _device("lmbp_fit_objective", theta, J), stream, _ACT[act], _OBJ[objective],
            int(k), float(eps), theta.data_ptr(), J.data_ptr(), n)
    return J


def fit_anneal(act: str, k: int = 2, objective: str = "h", eps: float = 1e-8, chains: int = 148 * 128,
               iters: int = 3000, seed: int = 2406, t0: float = 0.1, t1: float = 1e-9, step0: float = 0.3,
               step1: float = 1e-9, init=None, device="cuda", stream=None, projected: bool = False):
    """Simulated annealing on the GPU, one chain per thread.  Returns
    (best [P + 1] = theta then J, chain_theta [chains, P], chain_J [chains]),
    all CUDA float64 tensors.  projected=True: lmbp_fit_anneal_vp (anneal
    the thresholds, weights by least squares)."""
    P = fit_n_params(k)
    if init is not None:
        _need(init, "init")
        if init.dtype != torch.float64 or init.numel() != P:
            raise ValueError(f"init must be float64 [{P}]")
    chain_theta = torch.empty(chains, P, dtype=torch.float64, device=device)
    chain_J = torch.empty(chains, dtype=torch.float64, device=device)
    best = torch.empty(P + 1, dtype=torch.float64, device=device)
    fn = "lmbp_fit_anneal_vp" if projected else "lmbp_fit_anneal"
    dev = _device(fn, chain_theta, *(() if init is None else (init,)))
    _launch(fn, dev, stream, _ACT[act], _OBJ[objective], int(k), float(eps),
            None if init is None else init.data_ptr(), int(chains), int(iters), int(seed) & (2 ** 64 - 1), float(t0),
            float(t1), float(step0), float(step1), chain_theta.data_ptr(), chain_J.data_ptr(), best.data_ptr())
    return best, chain_theta, chain_J


def fit_refine(theta, act: str, k: int = 2, objective: str = "h", eps: float = 1e-8, iters: int = 40, stream=None):
    """Levenberg-Marquardt refinement of every row of theta [n, P] (CUDA
    float64).  Returns (best [P + 1], theta_out [n, P], J_out [n])."""
    _need(theta, "theta")
    P = fit_n_params(k)
    if theta.dtype != torch.float64 or theta.dim() != 2 or theta.shape[1] != P:
        raise ValueError(f"theta must be float64 [n, {P}]")
    n = theta.shape[0]
    out = torch.empty_like(theta)
    J = torch.empty(n, dtype=torch.float64, device=theta.device)
    best = torch.empty(P + 1, dtype=torch.float64, device=theta.device)
    _launch("lmbp_fit_refine", theta.device, stream, _ACT[act], _OBJ[objective], int(k), float(eps),
            theta.data_ptr(), n, int(iters), out.data_ptr(), J.data_ptr(), best.data_ptr())
    return best, out, J
