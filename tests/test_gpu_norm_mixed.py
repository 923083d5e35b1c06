"""Mixed-precision MS-LN / MS-RMSNorm (fp32 residual stream, 16-bit y / dy;
the AMP layout of Fig. 5 / 6) against the float64 oracle:
forward y within the 16-bit bar of SURVEY 8(c) (rstd within fp32's), backward
dx (fp32) within the fp32 norm-backward bound on the same 16-bit (dy, y);
misaligned / ragged rows (scalar path) agree with the oracle too, and the
autograd module keeps exactly y (16-bit) + rstd."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2406_16282_b200 as P
from test_gpu_parity import ATOL, DEV, RTOL, dec, st

pytestmark = pytest.mark.gpu
OUT = {"bf16": torch.bfloat16, "f16": torch.float16}
FNS = {"ln": (P.msln_fwd_mixed, P.msln_bwd_mixed, oracle.msln_fwd, oracle.msln_bwd),
       "rms": (P.msrms_fwd_mixed, P.msrms_bwd_mixed, oracle.msrms_fwd, oracle.msrms_bwd)}


def run_case(norm, out, R, H, offset=0):
    nf, nb, of, ob = FNS[norm]
    x = synth.norm_input(R, H, "f32")
    dy = synth.grad_input(R, H, out, stream=synth.S_NORM_DY)
    xd = x.to(DEV)
    if offset:                                   # misaligned fp32 rows -> scalar path
        buf = torch.empty(R * H + offset, device=DEV)
        xd = buf[offset:].view(R, H)
        xd.copy_(x)
    y, rstd = nf(xd, 1e-6, OUT[out])
    torch.cuda.synchronize()
    x64 = x.double().numpy()
    y_ref, r_ref = of(x64, float(np.float32(1e-6)))
    r = rstd.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(r - r_ref) <= RTOL["f32"] * 4 * r_ref), "rstd"
    # LN: the computed mean carries a rounding error on the scale of the
    # summands, mean|x| (not |mean x|, which can be ~0 for a wide row)
    mu = np.abs(x64).mean(1, keepdims=True) if norm == "ln" else 0.0
    yg = dec(y, out)
    tol = RTOL[out] * (np.abs(y_ref) + r_ref[:, None] * mu) + ATOL[out]
    assert not (np.abs(yg - y_ref) > tol).any(), "y"
    dx = nb(dy.to(DEV), y, rstd)
    torch.cuda.synchronize()
    assert dx.dtype == torch.float32
    dy64 = dec(dy, out)
    ref = ob(dy64, yg, r)
    m1 = np.abs(dy64.mean(1, keepdims=True)) if norm == "ln" else 0.0
    scale = r[:, None] * (np.abs(dy64) + m1 + np.abs(yg) * np.abs(dy64 * yg).mean(1, keepdims=True))
    bad = np.abs(dx.cpu().double().numpy() - ref) > RTOL["f32"] * 4 * scale + ATOL["f32"]
    assert not bad.any(), f"dx: {bad.sum()} out of bound"


@pytest.mark.parametrize("norm", ["ln", "rms"])
@pytest.mark.parametrize("out", ["bf16", "f16"])
@pytest.mark.parametrize("H", [8, 64, 768, 1024, 1032, 4096, 5120, 16384])
def test_mixed_norm_vs_oracle(norm, out, H):
    run_case(norm, out, 37 if H <= 5120 else 3, H)


@pytest.mark.parametrize("norm", ["ln", "rms"])
@pytest.mark.parametrize("H", [7, 770, 20000])
def test_mixed_norm_scalar_paths(norm, H):
    run_case(norm, "bf16", 5, H)                      # cols % 8 != 0 or > 16384: scalar kernels
    run_case(norm, "bf16", 5, 768, offset=1)          # misaligned x


def test_mixed_module_saves_y16_and_rstd():
    R, H = 128, 768
    x = synth.norm_input(R, H, "f32").to(DEV).requires_grad_(True)
    m = P.MSLayerNorm(H, out_dtype=torch.bfloat16)
    lin = torch.nn.Linear(H, 64, bias=False, dtype=torch.bfloat16, device=DEV)
    both = P.saved_bytes(lambda t: lin(m(t)), x)
    assert both == R * H * 2 + 4 * R + H * 64 * 2        # bf16 y (shared with the linear) + rstd + weight
    y = m(x)
    assert y.dtype == torch.bfloat16
    g = synth.grad_input(R, H, "bf16").to(DEV)
    y.backward(g)
    y2, r2 = P.msln_fwd_mixed(x.detach(), 1e-6)
    assert x.grad.dtype == torch.float32
    assert torch.equal(x.grad, P.msln_bwd_mixed(g, y2, r2))
