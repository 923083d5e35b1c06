"""MS-LN / MS-RMSNorm at extreme row lengths (SURVEY 8(c) "maximum sizes"):
rows of 2^16 .. 2^20 (+ odd) elements, where the register teams give way to
the shared-memory ring and the scalar multi-pass CTA-per-row path, against
the float64 oracle with the DESIGN 7 bars; plus large-magnitude rows (values
~1e15 and ~1e-15, both far from the norm's eps) that stay inside binary32's
range for the sum of squares."""
import numpy as np
import pytest
import torch

import oracle
import synth
from test_gpu_parity import DEV, DT, NORM, check_norm_bwd, check_norm_fwd, dec

pytestmark = pytest.mark.gpu


def _run(norm, dtype, x, eps=1e-6):
    R, H = x.shape
    dy = synth.grad_input(R, H, dtype, stream=synth.S_NORM_DY)
    nf, nb, _, _ = NORM[norm]
    y, rstd = nf(x.to(DEV), eps)
    torch.cuda.synchronize()
    y_ref, r_ref = check_norm_fwd(norm, dtype, x, eps, y, rstd)
    y_in = synth.from_numpy_storage(oracle.round_to(y_ref, dtype), dtype).reshape(R, H)
    r_in = torch.from_numpy(r_ref.astype(np.float32))
    dx = nb(dy.to(DEV), y_in.to(DEV), r_in.to(DEV))
    torch.cuda.synchronize()
    check_norm_bwd(norm, dtype, dy, dec(y_in, dtype), r_in.numpy().astype(np.float64), dx)


@pytest.mark.parametrize("norm", ["ln", "rms"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("H", [65536, 65537, 262144, 1 << 20, (1 << 20) + 7])
def test_norm_long_rows(norm, dtype, H):
    x = synth.norm_input(2, H, dtype)
    _run(norm, dtype, x)


@pytest.mark.parametrize("norm", ["ln", "rms"])
@pytest.mark.parametrize("scale", [1e15, 1e-15])
def test_norm_large_and_small_magnitudes_f32(norm, scale):
    H = 4096
    x64 = synth.norm_input(3, H, "f32").double() * scale
    _run(norm, "f32", x64.float())
