"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests and
bench.py.  Holds NO arithmetic of the method: only shapes and random draws.

Recipe (the paper fixes no distributions, so these
are readings):

* activation input x (bench mode): N(0, 1) rounded to the storage type.  FFN
  pre-activations are roughly zero-mean, O(1).
* activation input x (coverage mode): 90 % N(0, 1) and 10 % U(-12, 12), so all
  four segments occur for SiLU too (its outer thresholds sit at about +-6.3,
  P:L1140).
* norm input x: row r is mu_r + sigma_r * N(0, 1), mu_r ~ U(-1, 1),
  sigma_r ~ U(0.5, 2) (per-token offset/scale of a residual stream).
* upstream gradients dy: N(0, 1).

Seeding is per 256-row block: block b of stream ``s`` uses the seed
``(base * 1_000_003 + s * 7_919 + b) mod 2^63``, so any row slice, generated on any
rank or device type, is bitwise identical to the same rows of the full tensor
*for a fixed device type* (CPU and CUDA generators differ; tests generate on
CPU and copy).

Configs C1..C5 mirror BASELINE.json "configs".
"""
from __future__ import annotations

import torch

BASE_SEED = 2406
BLOCK_ROWS = 256

# stream ids (keep different tensors independent)
S_ACT_X, S_ACT_DY, S_NORM_X, S_NORM_DY, S_NORM_Y, S_NORM_RSTD = 1, 2, 3, 4, 5, 6

TORCH_DTYPES = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
ELEM_BYTES = {"f32": 4, "bf16": 2, "f16": 2}

# name -> shapes.  R = tokens, F = activation width, H = normalised width.
CONFIGS = {
    "c1": dict(R=2 * 197, F=3072, H=768, dtype="f32", act="gelu", norm="ln", batch=2, seq=197, heads=12,
               desc="single ViT-B block slice: ReGELU2 on 2x197x3072 + MS-LN on 2x197x768, fp32",
               bj_index=0),
    "c2": dict(R=64 * 197, F=3072, H=768, dtype="bf16", act="gelu", norm="ln", batch=64, seq=197, heads=12,
               desc="ViT-B/16 LoRA: batch 64, 197 tokens, hidden 768, MLP 3072, bf16",
               bj_index=1),
    "c3": dict(R=32 * 512, F=3072, H=768, dtype="f32", act="gelu", norm="ln", batch=32, seq=512, heads=12,
               desc="RoBERTa-base: batch 32, seq 512, hidden 768, FFN 3072 (fp32, P:L734)",
               bj_index=2),
    "c4": dict(R=4 * 2048, F=11008, H=4096, dtype="bf16", act="silu", norm="rms", batch=4, seq=2048, heads=32,
               desc="LLaMA-7B: batch 4, seq 2048, hidden 4096, FFN 11008, ReSiLU2 gate + MS-RMSNorm, bf16",
               bj_index=3),
    "c5": dict(R=8 * 4096, F=13824, H=5120, dtype="bf16", act="silu", norm="rms", batch=8, seq=4096, heads=40,
               desc="LLaMA-13B: batch 8, seq 4096, hidden 5120, FFN 13824, ReSiLU2 + MS-RMSNorm, bf16",
               bj_index=4),
}


def _seed(stream: int, block: int, base: int = BASE_SEED) -> int:
    return (base * 1_000_003 + stream * 7_919 + block) % (1 << 63)


def _blocks(row_start: int, row_end: int):
    b0 = row_start // BLOCK_ROWS
    b1 = (row_end + BLOCK_ROWS - 1) // BLOCK_ROWS
    for b in range(b0, b1):
        lo = max(row_start, b * BLOCK_ROWS)
        hi = min(row_end, (b + 1) * BLOCK_ROWS)
        yield b, lo - b * BLOCK_ROWS, hi - b * BLOCK_ROWS, lo - row_start, hi - row_start


def _fill(out: torch.Tensor, row_start: int, cols: int, stream: int, draw, base: int):
    """Fill out[rows, cols] block by block; draw(gen, nrows) -> fp32 [nrows, cols]."""
    rows = out.shape[0]
    dev = out.device
    for b, blo, bhi, olo, ohi in _blocks(row_start, row_start + rows):
        g = torch.Generator(device=dev)
        g.manual_seed(_seed(stream, b, base))
        full = draw(g, BLOCK_ROWS)                     # whole block, then slice:
        out[olo:ohi].copy_(full[blo:bhi])              # slice-invariant by design
    return out


def act_input(rows: int, cols: int, dtype: str, *, row_start: int = 0, mode: str = "bench",
              device="cpu", base: int = BASE_SEED, stream: int = S_ACT_X) -> torch.Tensor:
    out = torch.empty(rows, cols, dtype=TORCH_DTYPES[dtype], device=device)

    def draw(g, n):
        z = torch.randn(n, cols, generator=g, device=out.device, dtype=torch.float32)
        if mode == "coverage":
            u = torch.rand(n, cols, generator=g, device=out.device, dtype=torch.float32)
            wide = torch.rand(n, cols, generator=g, device=out.device, dtype=torch.float32) * 24 - 12
            z = torch.where(u < 0.1, wide, z)
        return z
    return _fill(out, row_start, cols, stream, draw, base)


def grad_input(rows: int, cols: int, dtype: str, *, row_start: int = 0, device="cpu",
               base: int = BASE_SEED, stream: int = S_ACT_DY) -> torch.Tensor:
    out = torch.empty(rows, cols, dtype=TORCH_DTYPES[dtype], device=device)

    def draw(g, n):
        return torch.randn(n, cols, generator=g, device=out.device, dtype=torch.float32)
    return _fill(out, row_start, cols, stream, draw, base)


def norm_input(rows: int, cols: int, dtype: str, *, row_start: int = 0, device="cpu",
               base: int = BASE_SEED, stream: int = S_NORM_X) -> torch.Tensor:
    out = torch.empty(rows, cols, dtype=TORCH_DTYPES[dtype], device=device)

    def draw(g, n):
        mu = torch.rand(n, 1, generator=g, device=out.device) * 2 - 1
        sd = torch.rand(n, 1, generator=g, device=out.device) * 1.5 + 0.5
        z = torch.randn(n, cols, generator=g, device=out.device, dtype=torch.float32)
        return mu + sd * z
    return _fill(out, row_start, cols, stream, draw, base)


def rstd_input(rows: int, *, row_start: int = 0, device="cpu", base: int = BASE_SEED) -> torch.Tensor:
    """Positive fp32 per-row scales in [0.5, 2] (stand-in saved rstd for
    backward-only parity cases)."""
    out = torch.empty(rows, 1, dtype=torch.float32, device=device)

    def draw(g, n):
        return torch.rand(n, 1, generator=g, device=out.device) * 1.5 + 0.5
    return _fill(out, row_start, 1, S_NORM_RSTD, draw, base).reshape(rows)


def to_numpy_storage(t: torch.Tensor):
    """torch tensor -> numpy storage array in the oracle's convention
    (bf16 as uint16 bit patterns).  Plumbing only."""
    t = t.detach().contiguous().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().view("uint16")
    return t.numpy()


def from_numpy_storage(a, dtype: str) -> torch.Tensor:
    import numpy as np
    a = np.ascontiguousarray(a)
    if dtype == "bf16":
        return torch.from_numpy(a.view(np.int16).copy()).view(torch.bfloat16)
    return torch.from_numpy(a.copy())


def codes_input(n: int, *, device="cpu", base: int = BASE_SEED) -> torch.Tensor:
    """Uniformly random packed 2-bit codes for n elements (ceil(n/4) bytes),
    unused trailing bits zero -- a backward-only parity input."""
    nbytes = (int(n) + 3) // 4
    g = torch.Generator(device="cpu")
    g.manual_seed(_seed(7, 0, base))
    b = torch.randint(0, 256, (nbytes,), generator=g, dtype=torch.int32).to(torch.uint8)
    if n % 4 and nbytes:
        b[-1] &= (1 << (2 * (n % 4))) - 1
    return b.to(device)


def all_patterns16(dtype: str, *, finite_only: bool = False, cols: int = 256) -> torch.Tensor:
    """Every bf16 / fp16 bit pattern once, in ascending pattern order, as a
    [rows, cols] tensor (65 536 elements; NaN and +-inf included unless
    finite_only, then the 256 (bf16) / 2 048 (fp16) all-ones-exponent
    patterns are dropped).  The exhaustive 16-bit parity input."""
    import numpy as np
    assert dtype in ("bf16", "f16")
    b = np.arange(1 << 16, dtype=np.uint32).astype(np.uint16)
    if finite_only:
        shift, emask = (7, 0xFF) if dtype == "bf16" else (10, 0x1F)
        b = b[((b >> shift) & emask) != emask]
    t = torch.from_numpy(b.view(np.int16).copy())
    t = t.view(torch.bfloat16) if dtype == "bf16" else t.view(torch.float16)
    return t.reshape(-1, cols).contiguous()
