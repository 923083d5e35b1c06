"""Exhaustive 16-bit parity: every bf16 / fp16 bit pattern -- 65 536 inputs,
NaN, +-inf, +-0 and the subnormals included -- through the CUDA path (C ABI)
against the float64 oracle.

A 16-bit storage type has only 65 536 values, so for these kernels the
elementwise parity can be checked on the whole input domain instead of a
sample (DESIGN 7):

* ReGELU2 / ReSiLU2 forward: codes bytewise for every pattern (NaN -> code 0,
  R8); y <= 1 ulp of RN_T(y_ref) for every finite pattern (DESIGN 7), and the
  number of outputs that are not the correctly rounded exact value (binary64
  oracle rounded once to T, here) is measured and bounded;
* backward: every dy pattern under each of the four codes, bitwise equal to
  the contract RN_T(RN32(dy * RN32(s[code]))) (R5; NaN in, NaN out);
* k-bit step activations (k = 1..4): codes bytewise, dx bitwise;
* fused ReSwiGLU2: every finite gate pattern (codes bytewise, a within the
  act bar, dgate / dup bitwise to the composition contract).
"""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2406_16282_b200 as P
from paper_2406_16282_b200 import tables
from test_gpu_parity import ACT, DEV, RTOL, ATOL, bits, check_act_fwd, dec, st, ulp_dist

pytestmark = pytest.mark.gpu

DTYPES16 = ["bf16", "f16"]


def rn64_bits(v: np.ndarray, dtype: str):
    """binary64 -> T with ONE round-to-nearest-even (no binary32 step), as
    uint16 patterns, and the mask of values that are exactly a rounding
    midpoint of T in binary64 (there the binary64 oracle cannot decide the
    rounding: the exact value's excess over the midpoint is below its
    precision, e.g. GELU(x) = x/2 + 0.4 x^2 for a subnormal x).  Test-side
    reference for the correct-rounding count."""
    p, qmin = (8, -133) if dtype == "bf16" else (11, -24)  # significant bits, smallest quantum exponent
    v = np.asarray(v, dtype=np.float64)
    a = np.abs(v)
    _, e = np.frexp(a)                                      # a = m 2^e, 0.5 <= m < 1
    q = np.maximum(e - p, qmin)
    scaled = np.ldexp(a, -q)                                # exact
    tie = (scaled - np.floor(scaled)) == 0.5
    r = np.copysign(np.ldexp(np.rint(scaled), q), v)       # RNE; exactly representable in T
    with np.errstate(over="ignore"):
        if dtype == "f16":
            return r.astype(np.float16).view(np.uint16), tie
        return (r.astype(np.float32).view(np.uint32) >> 16).astype(np.uint16), tie


# Outputs that are not RN_T of the exact value, out of the finite patterns
# whose binary64 oracle value is not itself a rounding midpoint of T
# (measured on B200, profiles/r02/session4/exhaustive16.log).  The GELU
# forward of 16-bit types reads the correctly rounded table (lut.py): none.
# SiLU is evaluated in binary32 and rounded once more (DESIGN 5.1): the exact
# value lies within a binary32 rounding error of a T midpoint for bf16
# x = 2^-7 and -2^-8 (SiLU(x) = x/2 + x^2/4 - x^4/48, and x^2/4 is exactly
# half a T ulp of x/2 there) and for f16 x = 2^-24, -2.72, -4.92 -- each
# 1 ulp off, inside the bar.
MAX_NOT_RN = {("gelu", "bf16"): 0, ("gelu", "f16"): 0, ("silu", "bf16"): 2, ("silu", "f16"): 3}


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", DTYPES16)
def test_act_fwd_all_patterns(kind, dtype):
    x = synth.all_patterns16(dtype)
    fwd, _ = ACT[kind]
    y, codes = fwd(x.to(DEV))
    torch.cuda.synchronize()
    check_act_fwd(kind, dtype, x, y, codes)            # codes bytewise (all), y <= 1 ulp (finite)
    x64 = dec(x, dtype).reshape(-1)
    fin = np.isfinite(x64)
    y_ref, _ = oracle.act_fwd(kind, x64[fin])
    got = np.ascontiguousarray(st(y)).reshape(-1).view(np.uint16)[fin]
    want, tie = rn64_bits(y_ref, dtype)
    bad = (got != want) & ~tie
    not_rn = int(bad.sum())
    xb = np.ascontiguousarray(st(x)).reshape(-1).view(np.uint16)[fin]
    print(f"{kind}/{dtype}: {not_rn} of {int(fin.sum())} finite patterns not correctly rounded; "
          f"first (x, got, want): {[(hex(a), hex(b), hex(c)) for a, b, c in zip(xb[bad][:12], got[bad][:12], want[bad][:12])]}")
    assert not_rn <= MAX_NOT_RN[(kind, dtype)]


def _bwd_inputs(dtype):
    """Every dy pattern under each code 0..3: n = 4 x 65 536, codes[j] = j // 65 536."""
    dy = synth.all_patterns16(dtype)
    dy4 = torch.cat([dy] * 4)                                       # [1024, 256]
    codes = torch.repeat_interleave(torch.tensor([0x00, 0x55, 0xAA, 0xFF], dtype=torch.uint8), 65536 // 4)
    return dy4, codes


def _same_bits_or_both_nan(got_st, want_st, dtype):
    g, w = oracle.decode(got_st, dtype).reshape(-1), oracle.decode(want_st, dtype).reshape(-1)
    nan = np.isnan(w)
    assert np.array_equal(np.isnan(g), nan), "NaN positions differ"
    gb = np.ascontiguousarray(got_st).reshape(-1).view(np.uint16)[~nan]
    wb = np.ascontiguousarray(want_st).reshape(-1).view(np.uint16)[~nan]
    assert np.array_equal(gb, wb), f"{int((gb != wb).sum())} outputs not bitwise"


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", DTYPES16)
def test_act_bwd_all_patterns(kind, dtype):
    dy, codes = _bwd_inputs(dtype)
    _, bwd = ACT[kind]
    dx = bwd(dy.to(DEV), codes.to(DEV))
    torch.cuda.synchronize()
    want = oracle.act_bwd_contract(kind, codes.numpy(), st(dy), dtype)
    _same_bits_or_both_nan(st(dx), want, dtype)


def _kbit_tables(k):
    if k == 2:
        c, s = oracle.regelu2d_table()                 # the paper's ReGELU2-d (App. I)
        return list(c), list(s)
    rng = np.random.default_rng(100 + k)
    m = (1 << k) - 1
    return sorted((rng.normal(size=m) * 3).tolist()), rng.normal(size=m + 1).tolist()


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("act", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", DTYPES16)
def test_stepact_all_patterns(k, act, dtype):
    c, s = _kbit_tables(k)
    x = synth.all_patterns16(dtype)
    y, codes = P.stepact_fwd(x.to(DEV), act, k, c)
    torch.cuda.synchronize()
    x64 = dec(x, dtype).reshape(-1)
    y_ref, c_ref = oracle.stepact_fwd(act, k, c, x64)
    assert np.array_equal(codes.cpu().numpy(), c_ref), "codes differ"
    fin = np.isfinite(x64)
    yr = y_ref.reshape(-1)[fin]
    yg = dec(y, dtype).reshape(-1)[fin]
    assert np.all(np.abs(yg - yr) <= RTOL[dtype] * np.abs(yr) + ATOL[dtype])
    assert ulp_dist(st(y).reshape(-1)[fin], oracle.round_to(yr, dtype), dtype).max() <= 1
    # backward: every dy pattern under the oracle's codes of the same patterns
    dy = synth.all_patterns16(dtype)
    dx = P.stepact_bwd(dy.to(DEV), codes, k, s)
    torch.cuda.synchronize()
    want = oracle.stepact_bwd_contract(k, s, c_ref, st(dy), dtype)
    _same_bits_or_both_nan(st(dx), want, dtype)


@pytest.mark.parametrize("dtype", DTYPES16)
def test_stepact_k2_paper_tables_equal_specialised_all_patterns(dtype):
    x = synth.all_patterns16(dtype).to(DEV)
    for tab, fwd in ((tables.REGELU2, P.regelu2_fwd), (tables.RESILU2, P.resilu2_fwd)):
        y1, c1 = P.stepact_fwd(x, tab["act"], 2, tab["c"])
        y2, c2 = fwd(x)
        torch.cuda.synchronize()
        assert torch.equal(c1, c2)
        fin = torch.isfinite(x.float()).reshape(-1).cpu().numpy()
        assert np.array_equal(st(y1).reshape(-1)[fin], st(y2).reshape(-1)[fin])


@pytest.mark.parametrize("dtype", DTYPES16)
def test_reswiglu2_all_gate_patterns(dtype):
    from test_gpu_swiglu import run_case
    gate = synth.all_patterns16(dtype, finite_only=True)
    R, F = gate.shape
    up = synth.grad_input(R, F, dtype, stream=11).clamp(-1, 1)     # |a up| <= |a|: h stays finite
    dh = synth.grad_input(R, F, dtype, stream=12)
    run_case(R, F, dtype, gate=gate, up=up, dh=dh)
