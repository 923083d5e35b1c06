"""GPU parity for the fused ReSwiGLU2 kernels against
the float64 oracle: codes bytewise, a = SiLU(gate) within the act tolerance
(and <= 1 ulp for 16-bit types), h bitwise equal to the unfused composition
RN(a * up), backward (dgate, dup) bitwise equal to the oracle's composition
contract."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2406_16282_b200 as P
from test_gpu_parity import ATOL, DEV, RTOL, bits, dec, st, ulp_dist

pytestmark = pytest.mark.gpu

DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}


def run_case(R, F, dtype, gate=None, up=None, dh=None):
    gate = synth.act_input(R, F, dtype, mode="coverage") if gate is None else gate
    up = synth.grad_input(R, F, dtype, stream=11) if up is None else up
    dh = synth.grad_input(R, F, dtype, stream=12) if dh is None else dh
    h, a, codes = P.reswiglu2_fwd(gate.to(DEV), up.to(DEV))
    torch.cuda.synchronize()
    g64, u64 = dec(gate, dtype), dec(up, dtype)
    h_ref, a_ref, c_ref = oracle.reswiglu2_fwd(g64, u64)
    assert np.array_equal(codes.cpu().numpy(), c_ref), "codes"
    fin = np.isfinite(g64).reshape(-1)
    ag = dec(a, dtype).reshape(-1)[fin]
    ar = a_ref.reshape(-1)[fin]
    assert np.all(np.abs(ag - ar) <= RTOL[dtype] * np.abs(ar) + ATOL[dtype]), "a tolerance"
    if dtype != "f32":
        assert ulp_dist(st(a).reshape(-1)[fin], oracle.round_to(ar, dtype), dtype).max() <= 1
    comp = (a.float() * up.to(DEV).float()).to(DT[dtype])                 # unfused composition
    assert st(h).tobytes() == st(comp).tobytes(), "h != RN(a*up)"
    hr = h_ref.reshape(-1)[fin]
    hg = dec(h, dtype).reshape(-1)[fin]
    # h = RN(RN(a) up): the error of a (rtol |a| + atol, atol for subnormal a)
    # is scaled by |up| before h's own rounding
    ug = dec(up, dtype).reshape(-1)[fin]
    assert np.all(np.abs(hg - hr) <= 2 * RTOL[dtype] * np.abs(hr) + ATOL[dtype] * (1 + np.abs(ug))), "h tolerance"
    # backward on oracle-derived a (rounded to T) and the oracle's codes
    a_in = synth.from_numpy_storage(oracle.round_to(a_ref, dtype), dtype).reshape(R, F)
    dg, du = P.reswiglu2_bwd(dh.to(DEV), up.to(DEV), a_in.to(DEV), torch.from_numpy(c_ref).to(DEV))
    torch.cuda.synchronize()
    wdg, wdu = oracle.reswiglu2_bwd_contract(st(dh), st(up), st(a_in), c_ref, dtype)
    assert np.array_equal(bits(st(dg)), bits(wdg)), "dgate not bitwise"
    assert np.array_equal(bits(st(du)), bits(wdu)), "dup not bitwise"
    return h, a, codes, dg, du


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("shape", [(1, 1), (1, 5), (3, 7), (5, 33), (2, 4097), (37, 3072), (64, 11008)])
def test_reswiglu2_parity(dtype, shape):
    run_case(*shape, dtype)


@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_reswiglu2_misaligned_and_inplace(dtype):
    R, F = 9, 1000
    g = synth.act_input(R, F, dtype, mode="coverage").to(DEV)
    u = synth.grad_input(R, F, dtype, stream=11).to(DEV)
    dh = synth.grad_input(R, F, dtype, stream=12).to(DEV)
    h0, a0, c0 = P.reswiglu2_fwd(g, u)
    dg0, du0 = P.reswiglu2_bwd(dh, u, a0, c0)
    buf = torch.empty(R * F + 1, dtype=g.dtype, device=DEV)
    gm = buf[1:].view(R, F)
    gm.copy_(g)
    hm, am, cm = P.reswiglu2_fwd(gm, u)                       # scalar path
    cb = torch.empty(c0.numel() + 1, dtype=torch.uint8, device=DEV)
    cb[1:].copy_(c0)
    dgm, dum = P.reswiglu2_bwd(dh, u, a0, cb[1:])             # codes not 16B aligned -> scalar
    gi, ui = g.clone(), u.clone()
    P.reswiglu2_fwd(gi, ui, h=gi, a=ui)                       # outputs alias inputs
    torch.cuda.synchronize()
    assert st(h0).tobytes() == st(hm).tobytes() and st(a0).tobytes() == st(am).tobytes()
    assert torch.equal(c0, cm)
    assert st(dg0).tobytes() == st(dgm).tobytes() and st(du0).tobytes() == st(dum).tobytes()
    assert st(gi).tobytes() == st(h0).tobytes() and st(ui).tobytes() == st(a0).tobytes()


@pytest.mark.parametrize("cfg", ["c4", "c5"])
def test_reswiglu2_full_size_sampled(cfg):
    c = synth.CONFIGS[cfg]
    R, F, dtype = c["R"], c["F"], c["dtype"]
    if cfg == "c5":
        R //= 8
    g = synth.act_input(R, F, dtype, device=DEV)
    u = synth.grad_input(R, F, dtype, device=DEV, stream=11)
    dh = synth.grad_input(R, F, dtype, device=DEV, stream=12)
    h, a, codes = P.reswiglu2_fwd(g, u)
    dg, du = P.reswiglu2_bwd(dh, u, a, codes)
    torch.cuda.synchronize()
    rng = np.random.default_rng(1)
    rows = sorted(set([0, R - 1] + list(rng.choice(R, 40, replace=False))))
    idx = torch.tensor(rows, device=DEV)
    gs, us, dhs = g[idx].cpu(), u[idx].cpu(), dh[idx].cpu()
    h_ref, a_ref, c_ref = oracle.reswiglu2_fwd(dec(gs, dtype), dec(us, dtype))
    assert np.array_equal(codes.view(R, F // 4)[idx].cpu().numpy().reshape(-1), c_ref)
    ar = a_ref.reshape(-1)
    assert np.all(np.abs(dec(a[idx], dtype).reshape(-1) - ar) <= RTOL[dtype] * np.abs(ar) + ATOL[dtype])
    # backward contract on the GPU's own (a, codes) is a composition property:
    wdg, wdu = oracle.reswiglu2_bwd_contract(st(dhs), st(us), st(a[idx]), c_ref, dtype)
    assert np.array_equal(bits(st(dg[idx])), bits(wdg)) and np.array_equal(bits(st(du[idx])), bits(wdu))


def test_reswiglu2_module_saved_bytes():
    R, F = 64, 11008
    g = synth.act_input(R, F, "bf16").to(DEV).requires_grad_(True)
    u = synth.grad_input(R, F, "bf16", stream=11).to(DEV).requires_grad_(True)
    m = P.ReSwiGLU2()
    ours = P.saved_bytes(m, g, u)
    assert ours == 2 * R * F * 2 + oracle.codes_bytes(R * F)                # up + a + codes
    exact = P.saved_bytes(lambda x, y: torch.nn.functional.silu(x) * y, g, u)
    assert exact == 3 * R * F * 2                                          # gate + silu(gate) + up
    h = m(g, u)
    dh = synth.grad_input(R, F, "bf16", stream=12).to(DEV)
    h.backward(dh)
    _, a, c = P.reswiglu2_fwd(g.detach(), u.detach())
    dg, du = P.reswiglu2_bwd(dh, u.detach(), a, c)
    assert torch.equal(g.grad.view(torch.int16), dg.view(torch.int16))
    assert torch.equal(u.grad.view(torch.int16), du.view(torch.int16))
