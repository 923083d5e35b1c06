"""The 16-bit forward tables (paper_2406_16282_b200/lut.py, compiled into
liblmbp.so) are correctly rounded: RN_T(h(x)) for h = GELU / SiLU
(P:L349-350), checked on CPU against mpmath at 40 digits with an independent
rounding (nearest of the two neighbouring T values, ties to even) on a sample
of bit patterns that covers every exponent, subnormals and the tails."""
import math

import mpmath as mp
import numpy as np
import pytest
import torch

from paper_2406_16282_b200 import lut


def _ref_bits(act, fmt, bits):
    mp.mp.dps = 40
    dt = torch.bfloat16 if fmt == "bf16" else torch.float16
    x = float(torch.tensor([bits], dtype=torch.int32).to(torch.int16).view(dt).float())
    X = mp.mpf(x)
    exact = X * mp.ncdf(X) if act == "gelu" else X / (1 + mp.e ** (-X))
    # candidates: every T value adjacent to float(exact) (nextafter in T by bit stepping)
    t = torch.tensor([float(exact)], dtype=torch.float64).to(dt)
    b0 = int(t.view(torch.int16)) & 0xFFFF
    cands = []
    for db in (-2, -1, 0, 1, 2):
        b = (b0 + db) & 0xFFFF
        if ((b >> 15) ^ (b0 >> 15)) and b0 & 0x7FFF:           # do not wrap across the sign
            continue
        v = float(torch.tensor([b], dtype=torch.int32).to(torch.int16).view(dt).float())
        if np.isfinite(v):
            cands.append((abs(mp.mpf(v) - exact), b & 1, v, b))
    cands.sort()
    best = cands[0]
    if len(cands) > 1 and cands[1][0] == best[0]:               # exact tie: even significand
        best = min(cands[:2], key=lambda c: c[1])
    v, b = best[2], best[3]
    if v == 0.0:                                                # signed zero follows the sign of h(x)
        b = 0x8000 if exact < 0 or (exact == 0 and math.copysign(1.0, x) < 0) else 0
    return b


@pytest.mark.parametrize("act", ["gelu", "silu"])
@pytest.mark.parametrize("fmt", ["bf16", "f16"])
def test_table_is_correctly_rounded(act, fmt):
    t = lut.table(act, fmt)
    rng = np.random.default_rng(7)
    sample = set(rng.integers(0, 65536, 600).tolist())
    sample |= {0x0000, 0x8000, 0x0001, 0x8001, 0x0002, 0x0080 if fmt == "bf16" else 0x0400}
    x = lut.inputs(fmt)
    for b in sorted(sample):
        if not np.isfinite(x[b]):
            continue
        want = _ref_bits(act, fmt, b)
        assert int(t[b]) == want, (act, fmt, hex(b), x[b], hex(int(t[b])), hex(want))


def test_table_specials():
    for fmt in ("bf16", "f16"):
        x = lut.inputs(fmt)
        for act in ("gelu", "silu"):
            t = lut.table(act, fmt)
            pinf = int(np.where(np.isposinf(x))[0][0])
            ninf = int(np.where(np.isneginf(x))[0][0])
            assert t[pinf] == pinf                                # h(+inf) = +inf
            assert t[ninf] == 0x8000                              # h(-inf) -> -0
            nan = np.isnan(x)
            assert (t[nan] == (0x7FC0 if fmt == "bf16" else 0x7E00)).all()
