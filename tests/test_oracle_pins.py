"""Pins for the float64 oracle (oracle/) against things other than itself:
the paper's printed constants (tests/golden/), SPEC's worked examples,
high-precision mpmath evaluations of the paper's own formulas, exact rational
arithmetic, torch float64 autograd of the textbook LayerNorm/RMSNorm,
central finite differences, closed forms and invariants.

Each pin is chosen so a plausible oracle mistake (dropped term, wrong sign or
index, transposed operand, swapped constant, off-by-one in packing) fails it.
"""
import json
import math
import os
from fractions import Fraction

import mpmath
import numpy as np
import pytest
import torch

import oracle

GOLD = os.path.join(os.path.dirname(__file__), "golden")
mpmath.mp.dps = 50


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


PAPER = _load("paper_constants.json")
SPEC = _load("spec_examples.json")


# --------------------------------------------------------------------------
# constants and the step table
# --------------------------------------------------------------------------
@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_constants_match_paper_text(kind):
    c, s, a = oracle.step_table(kind)
    g = PAPER[kind]
    assert [float(v) for v in g["a"]] == list(a)
    assert [float(v) for v in g["c"]] == list(c)
    # the 4-significant-figure values of Sec. 4.2 are roundings of the full ones
    for full, short in zip(list(a) + list(c), g["a_short"] + g["c_short"]):
        digits = len(short.lstrip("-0.").replace(".", ""))
        assert float(f"{full:.{digits}g}") == float(short)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_levels_are_slopes_of_eq14(kind):
    """s[code] must equal the finite-difference slope of h~ (Eq. 14, written
    out independently here) inside each segment; s0=0 and s3=1 exactly."""
    c, s, a = oracle.step_table(kind)
    assert s[0] == 0.0 and s[3] == 1.0
    w = [a[0], a[1], 1.0 - a[0] - a[1]]

    def htilde(x):  # Eq. 14, k = 2
        return sum(wi * max(x - ci, 0.0) for wi, ci in zip(w, c))

    mids = [c[0] - 5.0, 0.5 * (c[0] + c[1]), 0.5 * (c[1] + c[2]), c[2] + 5.0]
    h = 1e-6
    for k, x in enumerate(mids):
        slope = (htilde(x + h) - htilde(x - h)) / (2 * h)
        assert abs(slope - s[k]) < 1e-8, (k, slope, s[k])
        _, codes = oracle.act_fwd(kind, np.array([x]))
        assert codes[0] == k
        # the oracle's own h~ agrees with the retyped Eq. 14
        assert abs(oracle.combo_eval(kind, x) - htilde(x)) < 1e-14 * (1 + abs(x))


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_eq14_constraint_and_limit(kind):
    """Eq. 14 constraint sum_i w_i c_i = 0 holds for the published constants
    (residual ~1e-16), hence h~(x) = x for x > c3 (Prop. 4.1.1)."""
    c, s, a = oracle.step_table(kind)
    w = [a[0], a[1], 1.0 - a[0] - a[1]]
    resid = sum(Fraction(wi) * Fraction(ci) for wi, ci in zip(w, c))
    assert abs(float(resid)) < 1e-12
    for x in (10.0, 50.0, 1e3):
        assert abs(oracle.combo_eval(kind, x) - x) < 1e-12 * x
    for x in (-10.0, -50.0):
        assert oracle.combo_eval(kind, x) == 0.0


def test_spec_level_examples():
    for ex in SPEC["codes"]:
        x = np.array([float(v) for v in ex["x"]])
        _, codes = oracle.act_fwd(ex["kind"], x)
        assert list(oracle.unpack_codes(codes, x.size)) == ex["codes"], ex["cite"]
        if "level" in ex:
            _, s, _ = oracle.step_table(ex["kind"])
            assert abs(s[ex["codes"][0]] - float(ex["level"])) <= 4e-16, ex["cite"]


# --------------------------------------------------------------------------
# exact forward against mpmath on the paper's formulas
# --------------------------------------------------------------------------
def _mp_gelu(x):  # paper form: x/2 (1 + erf(x/sqrt 2)); 500 digits so
    with mpmath.workdps(500):  # 1 + erf does not cancel to 0 in the left tail
        x = mpmath.mpf(x)
        return +(x / 2 * (1 + mpmath.erf(x / mpmath.sqrt(2))))


def _mp_silu(x):  # x / (1 + e^{-x})
    x = mpmath.mpf(x)
    return x / (1 + mpmath.exp(-x))


GRID = sorted(set([float(v) for v in np.linspace(-40, 40, 321)] +
                  [-37.5, -13.2, -9.0, -5.5, -3.1858810036855245, -1e-3, -1e-9, 0.0,
                   1e-300, 1e-9, 1e-3, 0.5, 3.19, 6.3, 38.2]))


@pytest.mark.parametrize("kind,ref", [("gelu", _mp_gelu), ("silu", _mp_silu)])
def test_forward_vs_mpmath(kind, ref):
    x = np.array(GRID)
    y, _ = oracle.act_fwd(kind, x)
    for xi, yi in zip(x, y):
        r = ref(xi)
        err = abs(mpmath.mpf(yi) - r)
        # relative 1e-13 on the body; in the far tail the binary64 rounding of
        # x/sqrt2 is amplified ~2z^2 by erfc, so 1e-10 there (still 1e5 x finer
        # than the fp32 parity tolerance); below the normal range: underflow.
        rtol = 1e-13 if abs(xi) <= 8 else 1e-10
        assert err <= rtol * abs(r) or err < 2.0**-1022, (kind, xi, yi, r)


def test_forward_spec_examples_and_odd_identity():
    for ex in SPEC["gelu_at"]:
        assert oracle.gelu(float(ex["x"])) == pytest.approx(float(ex["y"]), rel=1e-15, abs=0), ex["cite"]
    for ex in SPEC["silu_at"]:
        assert oracle.silu(float(ex["x"])) == float(ex["y"]), ex["cite"]
    # h(x) - h(-x) = x for both (Phi(-x) = 1 - Phi(x), sigma(-x) = 1 - sigma(x))
    rng = np.random.default_rng(0)
    for x in rng.uniform(-20, 20, 200):
        assert oracle.gelu(x) - oracle.gelu(-x) == pytest.approx(x, rel=1e-14, abs=1e-14)
        assert oracle.silu(x) - oracle.silu(-x) == pytest.approx(x, rel=1e-14, abs=1e-14)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_exact_derivative_vs_mpmath_diff(kind):
    ref = _mp_gelu if kind == "gelu" else _mp_silu
    for x in (-6.0, -2.5, -0.3, 0.0, 0.7, 2.0, 5.0):
        d = float(mpmath.diff(ref, x))
        assert oracle.act_deriv(kind, x) == pytest.approx(d, rel=1e-12, abs=1e-15)
    for ex in SPEC["deriv_at"]:
        assert oracle.act_deriv(ex["kind"], float(ex["x"])) == float(ex["d"]), ex["cite"]


# --------------------------------------------------------------------------
# codes: exact-real threshold contract (reading R2), packing
# --------------------------------------------------------------------------
@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_codes_exact_against_decimal_thresholds(kind):
    """code = #{i : x > c_i} with c_i the paper's DECIMAL string, compared in
    exact rational arithmetic, for the fp32 / bf16 / fp16 neighbours of every
    threshold and a random sample."""
    dec = [Fraction(v) for v in PAPER[kind]["c"]]
    xs = []
    for cd in dec:
        f = np.float32(float(cd))
        for k in range(-3, 4):
            xs.append(float(np.nextafter(f, np.float32(np.inf * np.sign(k or 1)), dtype=np.float32))
                      if k else float(f))
            v = f
            for _ in range(abs(k)):
                v = np.nextafter(v, np.float32(np.inf if k > 0 else -np.inf), dtype=np.float32)
            xs.append(float(v))
        h = np.float16(float(cd))
        xs += [float(h), float(np.nextafter(h, np.float16(np.inf))), float(np.nextafter(h, np.float16(-np.inf)))]
        b = torch.tensor(float(cd), dtype=torch.bfloat16)
        bits = b.view(torch.int16).item()
        for d in (-1, 0, 1):
            xs.append(torch.tensor(bits + d, dtype=torch.int16).view(torch.bfloat16).float().item())
    xs += list(np.random.default_rng(1).normal(size=2000) * 4)
    x = np.array(xs)
    _, codes = oracle.act_fwd(kind, x)
    got = oracle.unpack_codes(codes, x.size)
    want = [sum(Fraction(float(v)) > cd for cd in dec) for v in x]
    assert list(got) == want


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_codes_at_kink_take_lower_segment(kind):
    """x == c_i exactly (the binary64 constant) -> code i (strict '>')."""
    c, _, _ = oracle.step_table(kind)
    _, codes = oracle.act_fwd(kind, np.array(c))
    assert list(oracle.unpack_codes(codes, 3)) == [0, 1, 2]


def test_codes_nan_inf_and_monotone():
    x = np.array([np.nan, -np.inf, np.inf, -0.0, 0.0])
    _, codes = oracle.act_fwd("gelu", x)
    assert list(oracle.unpack_codes(codes, 5)) == [0, 0, 3, 2, 2]
    xs = np.sort(np.random.default_rng(2).normal(size=5000) * 8)
    for kind in ("gelu", "silu"):
        _, c = oracle.act_fwd(kind, xs)
        u = oracle.unpack_codes(c, xs.size)
        assert np.all(np.diff(u.astype(int)) >= 0)


def test_packing_layout():
    # [0,1,2,3] -> 0xE4: x chosen one per segment
    _, codes = oracle.act_fwd("gelu", np.array([-10.0, -1.0, 1.0, 10.0]))
    assert list(codes) == SPEC["pack"][0]["bytes"]
    _, codes = oracle.act_fwd("gelu", np.zeros(0))
    assert codes.size == 0
    # ragged tail: trailing bits zero, byte count ceil(n/4)
    for n in range(1, 13):
        x = np.full(n, 10.0)                                          # all code 3
        _, codes = oracle.act_fwd("silu", x)
        assert codes.size == (n + 3) // 4 == oracle.codes_bytes(n)
        full = n // 4
        assert all(b == 0xFF for b in codes[:full])
        if n % 4:
            assert codes[-1] == (1 << (2 * (n % 4))) - 1
    # round trip on random codes: pack by hand (independent of the oracle)
    rng = np.random.default_rng(3)
    cvals = rng.integers(0, 4, size=1001)
    packed = np.zeros((1001 + 3) // 4, dtype=np.uint8)
    for j, v in enumerate(cvals):
        packed[j // 4] |= np.uint8(v << (2 * (j % 4)))
    assert np.array_equal(oracle.unpack_codes(packed, 1001), cvals)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
def test_code_frequencies_under_normal(kind):
    """Under x ~ N(0,1) the code frequencies are differences of the normal CDF
    at the thresholds (closed form)."""
    from scipy.stats import norm
    c, _, _ = oracle.step_table(kind)
    n = 400_000
    x = np.random.default_rng(4).normal(size=n)
    _, codes = oracle.act_fwd(kind, x)
    freq = np.bincount(oracle.unpack_codes(codes, n), minlength=4) / n
    cdf = norm.cdf(c)
    want = np.array([cdf[0], cdf[1] - cdf[0], cdf[2] - cdf[1], 1 - cdf[2]])
    assert np.all(np.abs(freq - want) < 5 * np.sqrt(want * (1 - want) / n) + 1e-6)


# --------------------------------------------------------------------------
# act backward
# --------------------------------------------------------------------------
def test_act_bwd_examples():
    dy = np.random.default_rng(5).normal(size=9)
    zeros = np.zeros((9 + 3) // 4, dtype=np.uint8)
    threes = np.full((9 + 3) // 4, 0xFF, dtype=np.uint8)
    for kind in ("gelu", "silu"):
        assert np.all(oracle.act_bwd(kind, zeros, dy) == 0)
        assert np.array_equal(oracle.act_bwd(kind, threes, dy), dy)
    ex = SPEC["backward"][0]
    code = np.array([ex["code"]], dtype=np.uint8)
    dx = oracle.act_bwd(ex["kind"], code, np.array([float(ex["dy"])]))
    assert dx[0] == pytest.approx(float(ex["dx"]), rel=4e-16), ex["cite"]
    # contract mode: 2 * RN32(a1 + a2) = 0x40063d22 as binary32
    dxc = oracle.act_bwd_contract("gelu", code, np.array([2.0], dtype=np.float32), "f32")
    assert dxc.view(np.uint32)[0] == 0x40063D22
    with pytest.raises(ValueError):
        oracle.act_bwd("gelu", code, np.zeros(5))


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_act_bwd_contract_matches_torch(dtype):
    """Contract mode RN_T(RN32(dy*RN32(s))) equals torch's own fp32 multiply
    followed by its RNE cast to the storage type (independent library)."""
    rng = np.random.default_rng(6)
    n = 20_000
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dtype]
    dy_t = torch.from_numpy(rng.normal(size=n) * np.exp(rng.uniform(-20, 20, n))).to(tdt)
    cvals = rng.integers(0, 4, size=n)
    packed = np.zeros((n + 3) // 4, dtype=np.uint8)
    np.bitwise_or.at(packed, np.arange(n) // 4, (cvals << (2 * (np.arange(n) % 4))).astype(np.uint8))
    for kind in ("gelu", "silu"):
        _, s, _ = oracle.step_table(kind)
        lv = torch.tensor(s, dtype=torch.float64).float()[torch.from_numpy(cvals)]
        want = (dy_t.float() * lv).to(tdt)
        dy_np = dy_t.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else dy_t.numpy()
        got = oracle.act_bwd_contract(kind, packed, dy_np, dtype)
        want_np = want.view(torch.int16).numpy().view(np.uint16) if dtype == "bf16" else want.numpy()
        assert np.array_equal(got.view(np.uint8), want_np.view(np.uint8))


def test_gradient_gap_diagnostic():
    """Relative gap ||(s - h')dy|| / ||h' dy|| is finite and < 0.5 for GELU
    under N(0,1); zero in both far tails."""
    x = np.random.default_rng(7).normal(size=20_000)
    _, codes = oracle.act_fwd("gelu", x)
    dy = np.ones_like(x)
    g_hat = oracle.act_bwd("gelu", codes, dy)
    g = np.array([oracle.act_deriv("gelu", v) for v in x])
    gap = np.linalg.norm(g_hat - g) / np.linalg.norm(g)
    assert 0.2 < gap < 0.5
    for v in (100.0, -100.0):
        xv = np.full(8, v)
        _, c = oracle.act_fwd("gelu", xv)
        assert np.allclose(oracle.act_bwd("gelu", c, np.ones(8)),
                           [oracle.act_deriv("gelu", v)] * 8, atol=1e-10)


# --------------------------------------------------------------------------
# storage conversions (plumbing used by contract mode) vs torch
# --------------------------------------------------------------------------
def test_decode_exhaustive_16bit():
    bits = np.arange(65536, dtype=np.uint32).astype(np.uint16)
    got = oracle.decode(bits, "bf16")
    want = torch.from_numpy(bits.view(np.int16).copy()).view(torch.bfloat16).double().numpy()
    assert np.array_equal(got, want, equal_nan=True)
    got = oracle.decode(bits.view(np.float16), "f16")
    want = torch.from_numpy(bits.view(np.float16).copy()).double().numpy()
    assert np.array_equal(got, want, equal_nan=True)


def test_round_to_matches_torch():
    rng = np.random.default_rng(8)
    u = rng.integers(0, 2**32, size=200_000, dtype=np.uint64).astype(np.uint32)
    f = u.view(np.float32)
    ties = (rng.integers(0, 2**16, 1000).astype(np.uint32) << 16) | 0x8000   # exact bf16 ties
    f = np.concatenate([f, ties.view(np.float32), np.array([0, -0.0, np.inf, -np.inf, 1e-45, 3e38],
                                                            dtype=np.float32)])
    f = f[~np.isnan(f)]
    tb = torch.from_numpy(f.copy()).to(torch.bfloat16).view(torch.int16).numpy().view(np.uint16)
    assert np.array_equal(oracle.round_to(f.astype(np.float64), "bf16"), tb)
    th = torch.from_numpy(f.copy()).to(torch.float16).numpy()
    assert np.array_equal(oracle.round_to(f.astype(np.float64), "f16").view(np.uint16), th.view(np.uint16))
    d = rng.normal(size=10000) * 10.0 ** rng.uniform(-40, 38, 10000)
    assert np.array_equal(oracle.round_to(d, "f32"), torch.from_numpy(d).float().numpy())


# --------------------------------------------------------------------------
# MS-LN / MS-RMSNorm (Alg. 2, Alg. 3)
# --------------------------------------------------------------------------
def _torch_ln(x, eps):
    return torch.nn.functional.layer_norm(x, (x.shape[-1],), eps=eps)


def _torch_rms(x, eps):
    return x * torch.rsqrt((x * x).mean(-1, keepdim=True) + eps)


@pytest.mark.parametrize("H", [1, 2, 3, 7, 64, 768])
@pytest.mark.parametrize("eps", [1e-6, 1e-3])
def test_msln_matches_torch_layernorm(H, eps):
    """Forward equals torch's LayerNorm (alpha=1, beta=0); backward from
    (y, rstd) equals torch autograd of LayerNorm from x."""
    rng = np.random.default_rng(H)
    x = rng.normal(size=(5, H)) * 3 + rng.uniform(-2, 2, (5, 1))
    dy = rng.normal(size=(5, H))
    y, rstd = oracle.msln_fwd(x, eps)
    xt = torch.tensor(x, requires_grad=True)
    yt = _torch_ln(xt, eps)
    yt.backward(torch.tensor(dy))
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-12, atol=1e-12)
    dx = oracle.msln_bwd(dy, y, rstd)
    ref = xt.grad.numpy()
    scale = np.abs(ref).max() + 1e-300
    assert np.abs(dx - ref).max() <= 1e-10 * scale + 1e-13


@pytest.mark.parametrize("H", [1, 2, 3, 7, 64, 768])
@pytest.mark.parametrize("eps", [1e-6, 1e-3])
def test_msrms_matches_torch_rmsnorm(H, eps):
    rng = np.random.default_rng(100 + H)
    x = rng.normal(size=(5, H)) * 2 + 0.5
    dy = rng.normal(size=(5, H))
    y, rstd = oracle.msrms_fwd(x, eps)
    xt = torch.tensor(x, requires_grad=True)
    yt = _torch_rms(xt, eps)
    yt.backward(torch.tensor(dy))
    assert np.allclose(y, yt.detach().numpy(), rtol=1e-13, atol=1e-14)
    dx = oracle.msrms_bwd(dy, y, rstd)
    assert np.abs(dx - xt.grad.numpy()).max() <= 1e-10 * np.abs(xt.grad.numpy()).max() + 1e-13


@pytest.mark.parametrize("norm", ["ln", "rms"])
def test_norm_bwd_finite_differences(norm):
    """Central finite differences of the oracle's own forward:
    L = sum(dy * y(x)); dL/dx_i ~ (L(x+h e_i) - L(x-h e_i)) / 2h."""
    fwd, bwd = (oracle.msln_fwd, oracle.msln_bwd) if norm == "ln" else (oracle.msrms_fwd, oracle.msrms_bwd)
    rng = np.random.default_rng(9)
    H, eps, h = 16, 1e-3, 1e-6
    x = rng.normal(size=(1, H))
    dy = rng.normal(size=(1, H))
    y, rstd = fwd(x, eps)
    dx = bwd(dy, y, rstd)
    fd = np.zeros(H)
    for i in range(H):
        xp, xm = x.copy(), x.copy()
        xp[0, i] += h
        xm[0, i] -= h
        fd[i] = (np.sum(dy * fwd(xp, eps)[0]) - np.sum(dy * fwd(xm, eps)[0])) / (2 * h)
    assert np.allclose(dx[0], fd, rtol=1e-6, atol=1e-7)


def test_msln_closed_forms():
    eps = 1e-6
    # constant row -> y = 0, rstd = 1/sqrt(eps); dx = rstd (dy - mean dy)
    x = np.full((1, 8), 0.37)
    y, rstd = oracle.msln_fwd(x, eps)
    assert np.all(np.abs(y) < 1e-9) and rstd[0] == pytest.approx(1 / math.sqrt(eps), rel=1e-12)
    dy = np.arange(8.0)[None]
    dx = oracle.msln_bwd(dy, np.zeros_like(dy), rstd)
    assert np.allclose(dx, rstd[0] * (dy - dy.mean()), rtol=1e-14)
    # [1, -1] with eps -> 0 -> [1, -1]
    y, _ = oracle.msln_fwd(np.array([[1.0, -1.0]]), 1e-300)
    assert np.allclose(y, [[1.0, -1.0]], rtol=1e-15)
    # invariants on random rows: mean(y)=0, mean(y^2)=var/(var+eps),
    # sum(dx)=0, y.dx = eps rstd^3 (y.dy)
    rng = np.random.default_rng(10)
    x = rng.normal(size=(20, 33)) * rng.uniform(0.1, 3, (20, 1)) + rng.uniform(-5, 5, (20, 1))
    eps = 1e-3
    y, rstd = oracle.msln_fwd(x, eps)
    var = x.var(axis=1)
    assert np.all(np.abs(y.mean(1)) < 1e-14 * 33)
    assert np.allclose((y * y).mean(1), var / (var + eps), rtol=1e-13)
    dy = rng.normal(size=x.shape)
    dx = oracle.msln_bwd(dy, y, rstd)
    assert np.all(np.abs(dx.sum(1)) < 1e-12 * np.abs(dx).sum(1))
    assert np.allclose((y * dx).sum(1), eps * rstd**3 * (y * dy).sum(1), rtol=1e-9, atol=1e-14)
    # p = 2: dx = +-eps rstd^3 (g1 - g2)/2
    x2 = rng.normal(size=(6, 2))
    dy2 = rng.normal(size=(6, 2))
    y2, r2 = oracle.msln_fwd(x2, eps)
    dx2 = oracle.msln_bwd(dy2, y2, r2)
    half = eps * r2**3 * (dy2[:, 0] - dy2[:, 1]) / 2
    assert np.allclose(dx2[:, 0], half, rtol=1e-8, atol=1e-15)
    assert np.allclose(dx2[:, 1], -half, rtol=1e-8, atol=1e-15)


def test_msrms_closed_forms():
    # x = 0 -> y = 0, rstd = 1/sqrt(eps); ones, eps -> 0: y = 1
    y, r = oracle.msrms_fwd(np.zeros((1, 4)), 1e-6)
    assert np.all(y == 0) and r[0] == pytest.approx(1e3, rel=1e-12)
    y, r = oracle.msrms_fwd(np.ones((1, 9)), 1e-300)
    assert np.allclose(y, 1.0, rtol=1e-15) and r[0] == pytest.approx(1.0, rel=1e-15)
    # p = 1: dx = eps rstd^3 dy
    rng = np.random.default_rng(11)
    eps = 1e-3
    x = rng.normal(size=(7, 1))
    dy = rng.normal(size=(7, 1))
    y, r = oracle.msrms_fwd(x, eps)
    dx = oracle.msrms_bwd(dy, y, r)
    assert np.allclose(dx[:, 0], eps * r**3 * dy[:, 0], rtol=1e-8, atol=1e-15)
    # y.dx = eps rstd^3 (y.dy)
    x = rng.normal(size=(10, 40))
    dy = rng.normal(size=(10, 40))
    y, r = oracle.msrms_fwd(x, eps)
    dx = oracle.msrms_bwd(dy, y, r)
    assert np.allclose((y * dx).sum(1), eps * r**3 * (y * dy).sum(1), rtol=1e-9, atol=1e-14)


def test_norm_shape_errors():
    with pytest.raises(ValueError):
        oracle.msln_bwd(np.zeros((2, 3)), np.zeros((2, 4)), np.ones(2))
    with pytest.raises(ValueError):
        oracle.msrms_bwd(np.zeros((2, 3)), np.zeros((2, 3)), np.ones(3))


# --------------------------------------------------------------------------
# a7: bytes saved (P:L214 unit model)
# --------------------------------------------------------------------------
def test_saved_bytes():
    for n in (0, 1, 3, 4, 5, 1_210_368, 90_177_536):
        assert oracle.codes_bytes(n) == -(-n // 4)
    b = oracle.act_saved_bytes(90_177_536, 2)                 # C4 SiLU gate, bf16
    assert b["exact"] == 8 * b["ours"]
    b = oracle.act_saved_bytes(1_210_368, 4)                  # C1 GELU, fp32
    assert b["exact"] == 16 * b["ours"]
    nb = oracle.norm_saved_bytes(8192, 4096, 4)
    assert nb["ours"] == 4 * 8192 and nb["exact"] == 8192 * 4096 * 4
    # Fig. 2 decoded unit model: ViT block 19 units with GELU 4
    # and 2 LayerNorms (fp32 inputs) 4 -> 21.05 % each
    assert round(100 * 4 / 19, 2) == 21.05
    assert round(100 * (13824 / 5120) / 21.8, 2) == 12.39 and round(100 * 4 / 21.8, 2) == 18.35


def test_tail_interval_examples():
    """App. E tail bounds reproduce SPEC's B values."""
    for ex in SPEC["tail_interval"]:
        eps = float(ex["eps"])
        B = math.sqrt(-2 * math.log(eps)) if ex["kind"] == "gelu" else -2 * math.log(eps / 2)
        assert B == pytest.approx(float(ex["B"]), abs=1e-4), ex["cite"]
        # the oracle's primitive really is below the bound beyond B
        f = oracle.gelu if ex["kind"] == "gelu" else oracle.silu
        assert abs(f(-B)) < 1 and abs(f(B) - B) < 1


# --------------------------------------------------------------------------
# ReSwiGLU2: SwiGLU gate with ReSiLU2
# --------------------------------------------------------------------------
def test_reswiglu2_matches_torch_autograd():
    """Forward = torch float64 SiLU(g)*u; du = autograd wrt u; dg = autograd
    of h~(g)*u with h~ the Eq. 14 ReLU combination written in torch (its
    derivative is the step function away from the kinks)."""
    rng = np.random.default_rng(12)
    n = 4000
    g = rng.normal(size=n) * 4
    u = rng.normal(size=n)
    dh = rng.normal(size=n)
    c, s, a = oracle.step_table("silu")
    g = g[np.min(np.abs(g[:, None] - c[None, :]), axis=1) > 1e-6]      # away from kinks
    n = g.size
    u, dh = u[:n], dh[:n]
    h, act, codes = oracle.reswiglu2_fwd(g, u)
    gt = torch.tensor(g, requires_grad=True)
    ut = torch.tensor(u, requires_grad=True)
    ht = torch.nn.functional.silu(gt) * ut
    assert np.allclose(h, ht.detach().numpy(), rtol=1e-14, atol=1e-300)
    assert np.allclose(act, torch.nn.functional.silu(gt).detach().numpy(), rtol=1e-14, atol=1e-300)
    ht.backward(torch.tensor(dh))
    w = [a[0], a[1], 1.0 - a[0] - a[1]]
    g2 = torch.tensor(g, requires_grad=True)
    ht2 = sum(wi * torch.relu(g2 - ci) for wi, ci in zip(w, c)) * torch.tensor(u)
    ht2.backward(torch.tensor(dh))
    dg, du = oracle.reswiglu2_bwd(dh, u, act, codes)
    assert np.allclose(du, ut.grad.numpy(), rtol=1e-14, atol=1e-300)
    assert np.allclose(dg, g2.grad.numpy(), rtol=1e-12, atol=1e-300)


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_reswiglu2_contract_matches_torch_composition(dtype):
    """Contract = torch's own unfused composition: da = (dh*u) rounded to T,
    dg = (da.float() * RN32(s)) rounded to T, du = (dh*a) rounded to T."""
    tdt = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}[dtype]
    rng = np.random.default_rng(13)
    n = 5000
    dh = torch.from_numpy(rng.normal(size=n)).to(tdt)
    u = torch.from_numpy(rng.normal(size=n) * 3).to(tdt)
    a = torch.from_numpy(rng.normal(size=n)).to(tdt)
    cvals = rng.integers(0, 4, size=n)
    packed = np.zeros((n + 3) // 4, dtype=np.uint8)
    np.bitwise_or.at(packed, np.arange(n) // 4, (cvals << (2 * (np.arange(n) % 4))).astype(np.uint8))
    _, s, _ = oracle.step_table("silu")
    lv = torch.tensor(s).float()[torch.from_numpy(cvals)]
    da = (dh.float() * u.float()).to(tdt)
    want_dg = (da.float() * lv).to(tdt)
    want_du = (dh.float() * a.float()).to(tdt)
    st = (lambda t: t.view(torch.int16).numpy().view(np.uint16)) if dtype == "bf16" else (lambda t: t.numpy())
    dg, du = oracle.reswiglu2_bwd_contract(st(dh), st(u), st(a), packed, dtype)
    assert np.array_equal(dg.view(np.uint8), st(want_dg).view(np.uint8))
    assert np.array_equal(du.view(np.uint8), st(want_du).view(np.uint8))


# --------------------------------------------------------------------------
# k-bit step activations
# --------------------------------------------------------------------------
def _pack_k(codes, k):
    out = np.zeros((len(codes) * k + 7) // 8, dtype=np.uint8)
    for j, c in enumerate(codes):
        out[(k * j) // 8] |= np.uint8(int(c) << ((k * j) % 8))
    return out


def test_stepact_k1_is_relu_derivative():
    """k = 1, c = [0], s = (0, 1): the step derivative is ReLU' (closed form)."""
    rng = np.random.default_rng(14)
    x = rng.normal(size=1001)
    dy = rng.normal(size=1001)
    y, codes = oracle.stepact_fwd("gelu", 1, [0.0], x)
    assert np.array_equal(codes, _pack_k((x > 0).astype(int), 1))
    assert np.array_equal(oracle.stepact_bwd(1, [0.0, 1.0], codes, dy), dy * (x > 0))
    assert np.allclose(y, [oracle.gelu(v) for v in x], rtol=0, atol=0)


def test_stepact_k4_codes_are_searchsorted():
    rng = np.random.default_rng(15)
    c = np.sort(rng.normal(size=15) * 3)
    x = np.concatenate([rng.normal(size=3000) * 4, c])          # incl. the kinks themselves
    _, codes = oracle.stepact_fwd("silu", 4, c, x)
    want = np.searchsorted(c, x, side="left")                    # #{i : c_i < x}
    assert np.array_equal(codes, _pack_k(want, 4))
    s = rng.normal(size=16)
    dy = rng.normal(size=x.size)
    assert np.array_equal(oracle.stepact_bwd(4, s, codes, dy), s[want] * dy)


def _pack_bits(codes, k):
    """Independent bit-stream packer: stream bit k*j + b = bit b of code j
    (LSB first), built as one Python integer, then cut into bytes."""
    acc = 0
    for j, c in enumerate(codes):
        acc |= int(c) << (k * j)
    return np.frombuffer(acc.to_bytes((len(codes) * k + 7) // 8, "little"), dtype=np.uint8)


def test_stepact_k3_hand_packed_stream():
    """k = 3: codes 0..7 of x placed between thresholds 0.5 .. 6.5; the 24-bit
    stream 111 110 101 100 011 010 001 000 (LSB first) is 0xFAC688, i.e. the
    bytes 88 C6 FA -- codes 2 and 5 straddle byte boundaries."""
    c = np.arange(7) + 0.5                                         # 0.5, 1.5, ..., 6.5
    x = np.arange(8, dtype=np.float64)                             # code j for x = j
    _, codes = oracle.stepact_fwd("gelu", 3, c, x)
    assert codes.tolist() == [0x88, 0xC6, 0xFA]
    s = np.arange(8) * 10.0
    assert oracle.stepact_bwd(3, s, codes, np.ones(8)).tolist() == [0, 10, 20, 30, 40, 50, 60, 70]
    # ragged tail: 3 elements = 9 bits -> 2 bytes, unused bits zero
    _, c3 = oracle.stepact_fwd("gelu", 3, c, np.array([7.0, 7.0, 7.0]))
    assert c3.tolist() == [0xFF, 0x01]


def test_stepact_k3_codes_are_searchsorted():
    rng = np.random.default_rng(17)
    c = np.sort(rng.normal(size=7) * 3)
    x = np.concatenate([rng.normal(size=3001) * 4, c, np.nextafter(c, np.inf), [np.nan, np.inf, -np.inf]])
    _, codes = oracle.stepact_fwd("silu", 3, c, x)
    want = np.searchsorted(c, x, side="left")                    # #{i : c_i < x}
    want[np.isnan(x)] = 0                                         # NaN > c is false (R8)
    assert np.array_equal(codes, _pack_bits(want, 3))
    s = rng.normal(size=8)
    dy = rng.normal(size=x.size)
    assert np.array_equal(oracle.stepact_bwd(3, s, codes, dy), s[want] * dy)
    for k in (1, 2, 4):                                           # the same packer agrees for byte-local k
        cc = np.sort(rng.normal(size=(1 << k) - 1))
        _, ck = oracle.stepact_fwd("silu", k, cc, x[:1000])
        assert np.array_equal(ck, _pack_bits(np.searchsorted(cc, x[:1000], side="left"), k))


def test_stepact_k2_equals_regelu2_and_resilu2():
    rng = np.random.default_rng(16)
    x = rng.normal(size=2001) * 5
    for kind in ("gelu", "silu"):
        c, s, _ = oracle.step_table(kind)
        y1, c1 = oracle.stepact_fwd(kind, 2, c, x)
        y2, c2 = oracle.act_fwd(kind, x)
        assert np.array_equal(c1, c2) and np.array_equal(y1, y2)
        dy = rng.normal(size=x.size)
        assert np.array_equal(oracle.stepact_bwd(2, s, c1, dy), oracle.act_bwd(kind, c2, dy))


def test_regelu2d_table_from_paper():
    """App. I constants typed in tests/golden; levels = slopes of Eq. 14 (FD);
    the paper's own ReGELU2-d solution violates the Eq. 14 constraint by
    ~7.9e-4 (derived; the derivative table does not depend on it)."""
    c, s = oracle.regelu2d_table()
    g = PAPER["gelu_d"]
    assert list(c) == [float(v) for v in g["c"]]
    a1, a2 = (float(v) for v in g["a"])
    w = [a1, a2, 1.0 - a1 - a2]

    def htilde(x):
        return sum(wi * max(x - ci, 0.0) for wi, ci in zip(w, c))
    mids = [c[0] - 1, 0.5 * (c[0] + c[1]), 0.5 * (c[1] + c[2]), c[2] + 1]
    for kk, xm in enumerate(mids):
        assert abs((htilde(xm + 1e-7) - htilde(xm - 1e-7)) / 2e-7 - s[kk]) < 1e-7
    resid = sum(Fraction(wi) * Fraction(ci) for wi, ci in zip(w, c))
    assert abs(float(resid) + 7.87e-4) < 1e-5
