"""Correctly rounded 16-bit activation tables for the ReGELU2 / ReSiLU2
forward (DESIGN 5.1): for every bf16 / fp16 bit pattern x, the table holds
RN_T(h(x)), h = GELU (x Phi(x)) or SiLU (x / (1 + e^-x)).

A 16-bit input has only 65536 values, so the forward of a 16-bit tensor is a
lookup (one shared-memory load per element) instead of ~14 issue slots of
polynomial / MUFU math per element; the tables are build-time constants of the
library (generated here, compiled into liblmbp.so), like the step tables.

Values: float64 (scipy erfc / numpy exp, relative error ~1e-15), rounded to
T with round-to-nearest-even directly from binary64 (no double rounding
through binary32); any value within 2^-30 relative of a rounding midpoint of T
is recomputed with mpmath at 50 digits.  Subnormal outputs are kept (no
flush).  Non-finite inputs: NaN -> the canonical quiet NaN, +inf -> +inf,
-inf -> -0 (the limits; SURVEY Q8 excludes them from value parity).

Product code: shares nothing with oracle/ (which evaluates its own erfc /
exp in C).
"""
from __future__ import annotations

import math
import os

import numpy as np

FORMATS = {  # significant bits, min normal exponent, max finite
    "bf16": dict(p=8, emin=-126, emax=127),
    "f16": dict(p=11, emin=-14, emax=15),
}


def inputs(fmt: str) -> np.ndarray:
    """float64 values of all 65536 bit patterns (NaN for NaN patterns)."""
    b = np.arange(65536, dtype=np.uint32)
    with np.errstate(invalid="ignore"):   # the NaN patterns widen to NaN
        if fmt == "bf16":
            return (b << 16).astype(np.uint32).view(np.float32).astype(np.float64)
        return b.astype(np.uint16).view(np.float16).astype(np.float64)


def _gelu64(x: np.ndarray) -> np.ndarray:
    from scipy.special import erfc
    with np.errstate(all="ignore"):
        return 0.5 * x * erfc(-x / math.sqrt(2.0))


def _silu64(x: np.ndarray) -> np.ndarray:
    with np.errstate(all="ignore"):
        pos = x / (1.0 + np.exp(-x))
        ex = np.exp(np.minimum(x, 0.0))
        neg = x * ex / (1.0 + ex)
    return np.where(x >= 0, pos, neg)


def _mp(act: str, x: float):
    import mpmath as mp
    mp.mp.dps = 50
    X = mp.mpf(x)
    if act == "gelu":
        return X * mp.ncdf(X)
    return X / (1 + mp.e ** (-X))


def _round(v, fmt: str):
    """RNE of a binary64 value to the format.  Returns (rounded float,
    |fraction - 1/2| of v in units of the format's quantum at v)."""
    f = FORMATS[fmt]
    if v == 0.0:
        return v, 0.5
    m, e = math.frexp(abs(v))                         # |v| = m 2^e, 0.5 <= m < 1
    q_exp = max(e - f["p"], f["emin"] - f["p"] + 1)   # quantum 2^(e-p), or the subnormal quantum
    q = math.ldexp(abs(v), -q_exp)                    # exact (power-of-two scaling)
    fl = math.floor(q)
    frac = q - fl
    if frac > 0.5 or (frac == 0.5 and fl % 2 == 1):
        fl += 1
    return math.copysign(math.ldexp(fl, q_exp), v), abs(frac - 0.5)


def _round_mp(X, fmt: str) -> float:
    """RNE of an mpmath value to the format (exact arithmetic at 50 digits)."""
    import mpmath as mp
    f = FORMATS[fmt]
    if X == 0:
        return 0.0
    m, e = mp.frexp(abs(X))
    q_exp = max(int(e) - f["p"], f["emin"] - f["p"] + 1)
    q = mp.ldexp(abs(X), -q_exp)
    fl = int(mp.floor(q))
    frac = q - fl
    if frac > mp.mpf(0.5) or (frac == mp.mpf(0.5) and fl % 2 == 1):
        fl += 1
    return math.copysign(math.ldexp(fl, q_exp), float(X))


def _bits(r: float, fmt: str) -> int:
    if fmt == "bf16":
        b = int(np.array(r, dtype=np.float32).view(np.uint32))
        assert b & 0xFFFF == 0, (r, hex(b))     # exactly representable in bf16
        return b >> 16
    h = np.array(r, dtype=np.float16)
    assert float(h) == r, r
    return int(h.view(np.uint16))


def table(act: str, fmt: str) -> np.ndarray:
    """uint16[65536]: RN_fmt(act(x)) for every fmt bit pattern x."""
    x = inputs(fmt)
    v = _gelu64(x) if act == "gelu" else _silu64(x)
    f = FORMATS[fmt]
    maxf = (2.0 - 2.0 ** (1 - f["p"])) * 2.0 ** f["emax"]
    out = np.zeros(65536, dtype=np.uint16)
    nan_bits = 0x7FC0 if fmt == "bf16" else 0x7E00
    for i in range(65536):
        xi = x[i]
        if math.isnan(xi):
            out[i] = nan_bits
            continue
        if math.isinf(xi):
            out[i] = _bits(math.inf if xi > 0 else -0.0, fmt)
            continue
        vi = float(v[i])
        r, dist = _round(vi, fmt)
        if dist < 2.0 ** -24:                   # within ~1e-7 quanta of a midpoint: decide with 50 digits
            r = _round_mp(_mp(act, xi), fmt)
        if abs(r) > maxf:
            r = math.copysign(math.inf, r)
        out[i] = _bits(r if r != 0.0 else math.copysign(0.0, vi), fmt)
    return out


TABLES = [("gelu", "bf16"), ("silu", "bf16"), ("gelu", "f16"), ("silu", "f16")]


def c_name(act: str, fmt: str) -> str:
    return f"kLut{act.capitalize()}{'Bf16' if fmt == 'bf16' else 'F16'}"


def write_inc(path: str) -> None:
    """Write the four tables as a C++ include (device constants)."""
    lines = ["// generated by paper_2406_16282_b200/lut.py -- do not edit", "#pragma once", "#include <cstdint>",
             "namespace lmbp {"]
    for act, fmt in TABLES:
        t = table(act, fmt)
        lines.append(f"__device__ __align__(16) const uint16_t {c_name(act, fmt)}[65536] = {{")
        for r in range(0, 65536, 16):
            lines.append(",".join(f"0x{int(v):04x}" for v in t[r:r + 16]) + ",")
        lines.append("};")
    lines.append("}  // namespace lmbp")
    tmp = path + ".tmp"
    with open(tmp, "w") as f:
        f.write("\n".join(lines) + "\n")
    os.replace(tmp, path)


if __name__ == "__main__":
    import sys
    write_inc(sys.argv[1])
