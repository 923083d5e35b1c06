"""Edge cases of the TMA/CLC pipeline (ew_pipeline.cuh): element counts at and
around tile boundaries (forward tile 1024 vectors, backward tile 1536 vectors,
the leftover pseudo-tile and the ragged element tail), and concurrent launches
on several streams (work stealing is per grid)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2406_16282_b200 as P
from test_gpu_parity import DEV, check_act_bwd, check_act_fwd, st, ulp_dist

pytestmark = pytest.mark.gpu

VEC = {"f32": 4, "bf16": 8}


def sizes(dtype):
    v = VEC[dtype]
    out = []
    for tile in (1024, 1536):
        for k in (1, 2, 3):
            base = tile * v * k
            out += [base, base + v, base + 1, base - 1, base - v, base + 3 * v + 5]
    return sorted(set(n for n in out if n > 0))


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_tile_boundaries(kind, dtype):
    fwd, bwd = (P.regelu2_fwd, P.regelu2_bwd) if kind == "gelu" else (P.resilu2_fwd, P.resilu2_bwd)
    for n in sizes(dtype):
        x = synth.act_input(1, n, dtype, mode="coverage")
        dy = synth.grad_input(1, n, dtype)
        y, codes = fwd(x.to(DEV))
        torch.cuda.synchronize()
        c_ref = check_act_fwd(kind, dtype, x, y, codes)
        dx = bwd(dy.to(DEV), torch.from_numpy(c_ref).to(DEV))
        torch.cuda.synchronize()
        check_act_bwd(kind, dtype, c_ref, dy, dx)


def test_reswiglu2_tile_boundaries():
    for n in sizes("bf16"):
        g = synth.act_input(1, n, "bf16", mode="coverage").to(DEV)
        u = synth.grad_input(1, n, "bf16", stream=11).to(DEV)
        h, a, c = P.reswiglu2_fwd(g, u)
        _, c_ref = oracle.act_fwd("silu", oracle.decode(st(g), "bf16"))
        torch.cuda.synchronize()
        assert np.array_equal(c.cpu().numpy(), c_ref)
        comp = (a.float() * u.float()).to(torch.bfloat16)
        assert torch.equal(h.view(torch.int16), comp.view(torch.int16))


def test_concurrent_streams_match_serial():
    xs = [synth.act_input(64, 11008, "bf16", row_start=64 * i).to(DEV) for i in range(4)]
    serial = [P.resilu2_fwd(x) for x in xs]
    torch.cuda.synchronize()
    streams = [torch.cuda.Stream() for _ in xs]
    outs = []
    for x, s in zip(xs, streams):
        with torch.cuda.stream(s):
            outs.append(P.resilu2_fwd(x, stream=s))
    torch.cuda.synchronize()
    for (y0, c0), (y1, c1) in zip(serial, outs):
        assert torch.equal(c0, c1) and torch.equal(y0.view(torch.int16), y1.view(torch.int16))


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_stepact_tile_boundaries(kind, k):
    """k-bit forwards on 16-bit types at and around their tile sizes: the
    GELU table shape (1024 vectors), the SiLU code-table shape (768 vectors),
    the backward (1536); codes bytewise and dx bitwise against the oracle."""
    m = (1 << k) - 1
    thr = [-3.0 + 6.0 * i / (m - 1) for i in range(m)]
    lv = [(-1) ** i * (i + 1) / m for i in range(m + 1)]
    out = []
    for tile in (768, 1024, 1536):
        for j in (1, 2):
            base = tile * 8 * j
            out += [base, base + 8, base + 1, base - 1, base - 8, base + 3 * 8 + 5]
    for n in sorted(set(out)):
        x = synth.act_input(1, n, "bf16", mode="coverage")
        dy = synth.grad_input(1, n, "bf16")
        y, codes = P.stepact_fwd(x.to(DEV), kind, k, thr)
        dx = P.stepact_bwd(dy.to(DEV), codes, k, lv)
        torch.cuda.synchronize()
        x64 = oracle.decode(st(x), "bf16")
        y_ref, c_ref = oracle.stepact_fwd(kind, k, thr, x64)
        assert np.array_equal(codes.cpu().numpy(), c_ref), (kind, k, n)
        want = oracle.stepact_bwd_contract(k, lv, c_ref, st(dy), "bf16")
        assert np.array_equal(st(dx).view(np.uint16), want.view(np.uint16)), (kind, k, n)
        yr = oracle.round_to(y_ref.reshape(-1), "bf16")
        d = ulp_dist(st(y).reshape(-1), yr, "bf16")
        finite = np.isfinite(x64.reshape(-1))
        assert d[finite].max() <= 1, (kind, k, n)
