"""GPU parity for the table-driven k-bit step activations (SURVEY 8(f)
NEXT #3): k = 2 with the published tables is bitwise identical to the
specialised regelu2/resilu2 kernels; k = 1, 2 (ReGELU2-d), 3, 4 against the
oracle (codes bytewise, y within tolerance, dx bitwise to the contract)."""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2406_16282_b200 as P
from paper_2406_16282_b200 import tables
from test_gpu_parity import ATOL, DEV, RTOL, bits, dec, st

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("shape", [(1, 3), (3, 7), (37, 3072), (5, 1001)])
def test_stepact_k2_paper_tables_equal_specialised(dtype, shape):
    x = synth.act_input(*shape, dtype, mode="coverage").to(DEV)
    dy = synth.grad_input(*shape, dtype).to(DEV)
    for tab, fwd, bwd in ((tables.REGELU2, P.regelu2_fwd, P.regelu2_bwd),
                          (tables.RESILU2, P.resilu2_fwd, P.resilu2_bwd)):
        y1, c1 = P.stepact_fwd(x, tab["act"], 2, tab["c"])
        y2, c2 = fwd(x)
        dx1 = P.stepact_bwd(dy, c1, 2, tables.levels(tab))
        dx2 = bwd(dy, c2)
        torch.cuda.synchronize()
        assert torch.equal(c1, c2)
        assert st(y1).tobytes() == st(y2).tobytes()
        assert st(dx1).tobytes() == st(dx2).tobytes()


def _tables(k, rng):
    if k == 1:
        return [0.0], [0.0, 1.0]
    if k == 2:
        c, s = oracle.regelu2d_table()
        return list(c), list(s)
    m = (1 << k) - 1
    c = sorted(rng.normal(size=m) * 3)
    return c, list(rng.normal(size=m + 1))


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("shape", [(1, 5), (7, 33), (64, 3072)])
def test_stepact_vs_oracle(k, dtype, shape):
    rng = np.random.default_rng(k)
    c, s = _tables(k, rng)
    x = synth.act_input(*shape, dtype, mode="coverage")
    dy = synth.grad_input(*shape, dtype)
    y, codes = P.stepact_fwd(x.to(DEV), "gelu", k, c)
    dx = P.stepact_bwd(dy.to(DEV), codes, k, s)
    torch.cuda.synchronize()
    x64 = dec(x, dtype)
    y_ref, c_ref = oracle.stepact_fwd("gelu", k, c, x64)
    assert np.array_equal(codes.cpu().numpy(), c_ref)
    yr = y_ref.reshape(-1)
    assert np.all(np.abs(dec(y, dtype).reshape(-1) - yr) <= RTOL[dtype] * np.abs(yr) + ATOL[dtype])
    want = oracle.stepact_bwd_contract(k, s, c_ref, st(dy), dtype)
    assert np.array_equal(bits(st(dx)), bits(want))


def test_stepact_bad_tables():
    x = torch.zeros(4, 8, device=DEV)
    with pytest.raises(RuntimeError, match="TABLE"):
        P.stepact_fwd(x, "gelu", 2, [1.0, 0.0, 2.0])           # not increasing
    with pytest.raises(RuntimeError, match="TABLE"):
        P.stepact_fwd(x, "gelu", 2, [0.0, float("nan"), 2.0])


@pytest.mark.parametrize("k", [1, 2, 3, 4])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_stepact_paths_bitwise(k, dtype):
    """TMA pipeline path (aligned) == simple kernel path (misaligned codes)."""
    rng = np.random.default_rng(10 + k)
    c, s = _tables(k, rng)
    R, F = 33, 4099
    x = synth.act_input(R, F, dtype, mode="coverage").to(DEV)
    dy = synth.grad_input(R, F, dtype).to(DEV)
    y0, c0 = P.stepact_fwd(x, "silu", k, c)
    dx0 = P.stepact_bwd(dy, c0, k, s)
    cb = torch.empty(c0.numel() + 1, dtype=torch.uint8, device=DEV)
    y1, c1 = P.stepact_fwd(x, "silu", k, c, codes=cb[1:])
    dx1 = P.stepact_bwd(dy, c1, k, s)
    torch.cuda.synchronize()
    assert torch.equal(c0, c1)
    assert st(y0).tobytes() == st(y1).tobytes() and st(dx0).tobytes() == st(dx1).tobytes()


@pytest.mark.parametrize("k", [3, 4])
@pytest.mark.parametrize("cfg", ["c3", "c4"])
def test_stepact_full_size_sampled(cfg, k):
    """k = 4 at the BASELINE config's full activation size (TMA/CLC pipeline,
    binary-search packed compares, shared-memory level table), sampled rows
    against the oracle: codes bytewise, y within tolerance, dx bitwise."""
    from test_gpu_parity import sample_rows
    c = synth.CONFIGS[cfg]
    R, F, dtype = c["R"], c["F"], c["dtype"]
    m = (1 << k) - 1
    thr = [-3.0 + 6.0 * i / (m - 1) for i in range(m)]
    lv = [(-1) ** i * i / m for i in range(m + 1)]
    x = synth.act_input(R, F, dtype, device=DEV, mode="coverage")
    dy = synth.grad_input(R, F, dtype, device=DEV)
    y, codes = P.stepact_fwd(x, c["act"], k, thr)
    dx = P.stepact_bwd(dy, codes, k, lv)
    torch.cuda.synchronize()
    rows = sample_rows(R)
    idx = torch.tensor(rows, device=DEV)
    assert (F * k) % 8 == 0                                     # a row's codes are whole bytes
    cb = codes.view(R, F * k // 8)[idx].cpu().numpy().reshape(-1)
    xs = x[idx].cpu()
    y_ref, c_ref = oracle.stepact_fwd(c["act"], k, thr, dec(xs, dtype))
    assert np.array_equal(cb, c_ref)
    yr = y_ref.reshape(-1)
    assert np.all(np.abs(dec(y[idx].cpu(), dtype).reshape(-1) - yr) <= RTOL[dtype] * np.abs(yr) + ATOL[dtype])
    want = oracle.stepact_bwd_contract(k, lv, c_ref, st(dy[idx].cpu()), dtype)
    assert np.array_equal(bits(st(dx[idx].cpu())), bits(want))


@pytest.mark.parametrize("act", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_stepact_k3_with_fitted_table(act, dtype):
    """The fitter's k = 3 solution (App. E objective, 7 ReLUs) fed straight
    into the k = 3 kernels: codes bytewise and dx bitwise against the oracle
    run with the same table; the table's levels are the Eq. 14 slopes."""
    from paper_2406_16282_b200 import fit as gfit
    f = gfit.fit(act, k=3, chains=2048, iters=800, refine_iters=10)
    tab = tables.from_fit(f)
    lv = tables.levels(tab)
    assert len(tab["c"]) == 7 and len(lv) == 8 and lv[0] == 0.0 and lv[-1] == 1.0
    R, F = 64, 3072 + 8 * 3 + 5                                 # ragged: a code straddles the last bytes
    x = synth.act_input(R, F, dtype, mode="coverage")
    dy = synth.grad_input(R, F, dtype)
    y, codes = P.stepact_fwd(x.to(DEV), act, 3, tab["c"])
    dx = P.stepact_bwd(dy.to(DEV), codes, 3, lv)
    torch.cuda.synchronize()
    y_ref, c_ref = oracle.stepact_fwd(act, 3, tab["c"], dec(x, dtype))
    assert np.array_equal(codes.cpu().numpy(), c_ref)
    want = oracle.stepact_bwd_contract(3, lv, c_ref, st(dy), dtype)
    assert np.array_equal(bits(st(dx)), bits(want))
    seg = np.bincount(np.searchsorted(np.array(tab["c"]), dec(x, dtype).reshape(-1), side="left"), minlength=8)
    assert (seg > 0).all(), seg
