"""GPU parity: the CUDA path (through the C ABI) against the float64 oracle on
the same seeded inputs.

Bars:
* codes: bytewise equal (BASELINE.json north_star "bit-exact 2-bit codes");
* act backward: bitwise equal to RN_T(RN32(dy * RN32(s[code]))) (reading R5);
* act forward y: |d| <= rtol |y| + atol, rtol = 1e-5 (fp32), 2e-2 (bf16)
  from north_star, 5e-3 (fp16, ours); plus <= 1 ulp of RN_T(y_ref) for bf16/fp16;
* norm forward: |dy_i| <= rtol (|y_i| + rstd |mu|) + atol; |d rstd| <= rtol rstd;
* norm backward: |d_i| <= rtol rstd (|dy_i| + |m1| + |y_i| mean|dy y|) + atol.
"""
import numpy as np
import pytest
import torch

import oracle
import synth
import paper_2406_16282_b200 as P

pytestmark = pytest.mark.gpu

RTOL = {"f32": 1e-5, "bf16": 2e-2, "f16": 5e-3}
ATOL = {"f32": 2.0 ** -126, "bf16": 2.0 ** -126, "f16": 2.0 ** -24}
DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
ACT = {"gelu": (P.regelu2_fwd, P.regelu2_bwd), "silu": (P.resilu2_fwd, P.resilu2_bwd)}
NORM = {"ln": (P.msln_fwd, P.msln_bwd, oracle.msln_fwd, oracle.msln_bwd),
        "rms": (P.msrms_fwd, P.msrms_bwd, oracle.msrms_fwd, oracle.msrms_bwd)}
DEV = "cuda"


def st(t):
    return synth.to_numpy_storage(t)


def dec(t, dtype):
    return oracle.decode(st(t), dtype)


def bits(a):
    return np.ascontiguousarray(a).view(np.uint8)


def ulp_dist(a_st, b_st, dtype):
    """|ordinal(a) - ordinal(b)| for 16-bit storage patterns."""
    a = np.ascontiguousarray(a_st).view(np.int16).astype(np.int32)
    b = np.ascontiguousarray(b_st).view(np.int16).astype(np.int32)
    a = np.where(a < 0, -32768 - a, a)
    b = np.where(b < 0, -32768 - b, b)
    return np.abs(a - b)


def check_act_fwd(kind, dtype, x_cpu, y_gpu, codes_gpu):
    x64 = dec(x_cpu, dtype)
    y_ref, c_ref = oracle.act_fwd(kind, x64)
    assert np.array_equal(codes_gpu.cpu().numpy(), c_ref), "codes differ"
    finite = np.isfinite(x64).reshape(-1)
    y = dec(y_gpu, dtype).reshape(-1)[finite]
    yr = y_ref.reshape(-1)[finite]
    err = np.abs(y - yr)
    bad = err > RTOL[dtype] * np.abs(yr) + ATOL[dtype]
    assert not bad.any(), (f"{kind}/{dtype}: {bad.sum()} y out of tol; worst x="
                           f"{x64.reshape(-1)[finite][bad][:5]}, y={y[bad][:5]}, ref={yr[bad][:5]}")
    if dtype != "f32":
        d = ulp_dist(st(y_gpu).reshape(-1)[finite], oracle.round_to(yr, dtype), dtype)
        assert d.max() <= 1, f"{kind}/{dtype}: {d.max()} ulp"
    return c_ref


def check_act_bwd(kind, dtype, codes_cpu_np, dy_cpu, dx_gpu):
    want = oracle.act_bwd_contract(kind, codes_cpu_np, st(dy_cpu), dtype)
    got = st(dx_gpu)
    assert np.array_equal(bits(got), bits(want)), f"{kind}/{dtype} act bwd not bitwise"


SHAPES = [(1, 1), (1, 3), (3, 7), (5, 33), (2, 4097), (37, 3072), (197, 768)]


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("shape", SHAPES)
def test_act_parity(kind, dtype, shape):
    R, F = shape
    x = synth.act_input(R, F, dtype, mode="coverage")
    dy = synth.grad_input(R, F, dtype)
    fwd, bwd = ACT[kind]
    y, codes = fwd(x.to(DEV))
    torch.cuda.synchronize()
    c_ref = check_act_fwd(kind, dtype, x, y, codes)
    # backward on the oracle's own codes (equal to the GPU's, checked above)
    dx = bwd(dy.to(DEV), torch.from_numpy(c_ref).to(DEV))
    torch.cuda.synchronize()
    check_act_bwd(kind, dtype, c_ref, dy, dx)
    # backward on independent random codes
    rc = synth.codes_input(R * F)
    dx2 = bwd(dy.to(DEV), rc.to(DEV))
    torch.cuda.synchronize()
    check_act_bwd(kind, dtype, rc.numpy(), dy, dx2)


def special_values(kind, dtype):
    c, _, _ = oracle.step_table(kind)
    vals = [0.0, -0.0, 88.0, -88.0, -87.5, -90.0, 100.0, -100.0, 1e4, -1e4, 13.2, -13.2, 6.0, -6.0,
            1e-30, -1e-30, 1e-40, -1e-40, 3e38, -3e38, 0.5, -0.5]
    for ci in c:
        f = np.float32(ci)
        for k in range(-2, 3):
            v = f
            for _ in range(abs(k)):
                v = np.nextafter(v, np.float32(np.inf if k > 0 else -np.inf), dtype=np.float32)
            vals.append(float(v))
        vals += [float(np.float16(ci)), float(torch.tensor(ci).to(torch.bfloat16).float())]
    return torch.tensor(vals, dtype=torch.float32).to(DT[dtype])


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_act_special_values(kind, dtype):
    x = special_values(kind, dtype)
    x = torch.cat([x, x.flip(0)])          # 2 rows of the same values, reversed
    x = x.reshape(2, -1).contiguous()
    y, codes = ACT[kind][0](x.to(DEV))
    torch.cuda.synchronize()
    check_act_fwd(kind, dtype, x, y, codes)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_act_nonfinite_codes(kind, dtype):
    """NaN -> code 0, -inf -> 0, +inf -> 3 (reading R8)."""
    x = torch.tensor([float("nan"), float("-inf"), float("inf"), 0.0, 1.0, -1.0, 2.0, -2.0, 5.0],
                     dtype=DT[dtype]).reshape(1, -1)
    y, codes = ACT[kind][0](x.to(DEV))
    _, c_ref = oracle.act_fwd(kind, dec(x, dtype))
    assert np.array_equal(codes.cpu().numpy(), c_ref)


@pytest.mark.parametrize("kind", ["gelu", "silu"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
def test_act_misaligned_and_inplace_bitwise(kind, dtype):
    """Scalar (misaligned) path == vector path bitwise; y == x in place ok."""
    R, F = 9, 1000
    x = synth.act_input(R, F, dtype, mode="coverage").to(DEV)
    dy = synth.grad_input(R, F, dtype).to(DEV)
    fwd, bwd = ACT[kind]
    y0, c0 = fwd(x)
    dx0 = bwd(dy, c0)
    buf = torch.empty(R * F + 1, dtype=x.dtype, device=DEV)
    xm = buf[1:].view(R, F)
    xm.copy_(x)                                    # 2-byte (or 4) offset: not 16B aligned
    ym, cm = fwd(xm)
    cbuf = torch.empty(c0.numel() + 1, dtype=torch.uint8, device=DEV)
    cmis = cbuf[1:]
    fwd(x, codes=cmis)                             # odd code pointer -> scalar path
    dxm = bwd(dy, cmis)
    xi = x.clone()
    fwd(xi, y=xi)                                  # in place
    dyi = dy.clone()
    bwd(dyi, c0, dx=dyi)
    torch.cuda.synchronize()
    assert st(y0).tobytes() == st(ym).tobytes()
    assert torch.equal(c0, cm) and torch.equal(c0, cmis)
    assert st(dx0).tobytes() == st(dxm).tobytes()
    assert st(xi).tobytes() == st(y0).tobytes()
    assert st(dyi).tobytes() == st(dx0).tobytes()


def test_act_deterministic_and_stream():
    x = synth.act_input(64, 3072, "bf16").to(DEV)
    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        y1, c1 = P.regelu2_fwd(x)
        y2, c2 = P.regelu2_fwd(x)
    s.synchronize()
    assert torch.equal(c1, c2) and torch.equal(y1.view(torch.int16), y2.view(torch.int16))


def test_act_empty():
    x = torch.empty(0, 16, device=DEV, dtype=torch.bfloat16)
    y, c = P.resilu2_fwd(x)
    assert y.numel() == 0 and c.numel() == 0


# ---------------------------------------------------------------------------
# norms
# ---------------------------------------------------------------------------
def check_norm_fwd(norm, dtype, x_cpu, eps, y_gpu, rstd_gpu):
    x64 = dec(x_cpu, dtype)
    eps32 = float(np.float32(eps))
    y_ref, r_ref = NORM[norm][2](x64, eps32)
    r = rstd_gpu.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(r - r_ref) <= RTOL[dtype] * r_ref), f"{norm}/{dtype} rstd"
    # LN: the computed mean carries a rounding error on the scale of the
    # summands, mean|x| (not |mean x|, which can be ~0 for a wide row)
    mu = np.abs(x64).mean(1, keepdims=True) if norm == "ln" else 0.0
    y = dec(y_gpu, dtype)
    tol = RTOL[dtype] * (np.abs(y_ref) + r_ref[:, None] * mu) + ATOL[dtype]
    bad = np.abs(y - y_ref) > tol
    assert not bad.any(), f"{norm}/{dtype}: {bad.sum()} y out of tol"
    return y_ref, r_ref


def check_norm_bwd(norm, dtype, dy_cpu, y_in64, rstd_in64, dx_gpu):
    dy64 = dec(dy_cpu, dtype)
    ref = NORM[norm][3](dy64, y_in64, rstd_in64)
    H = dy64.shape[1]
    m1 = np.abs(dy64.mean(1, keepdims=True)) if norm == "ln" else 0.0
    mdy = np.abs(dy64 * y_in64).mean(1, keepdims=True)
    scale = rstd_in64[:, None] * (np.abs(dy64) + m1 + np.abs(y_in64) * mdy)
    dx = dec(dx_gpu, dtype)
    bad = np.abs(dx - ref) > RTOL[dtype] * scale + ATOL[dtype]
    assert not bad.any(), f"{norm}/{dtype} H={H}: {bad.sum()} dx out of tol"
    rowerr = np.linalg.norm(dx - ref, axis=1)
    assert np.all(rowerr <= RTOL[dtype] * np.linalg.norm(scale, axis=1) + ATOL[dtype] * np.sqrt(H))


NORM_H = [1, 2, 3, 7, 8, 31, 32, 33, 127, 768, 1000, 1024, 3072, 4096, 5120, 11008, 40000]


@pytest.mark.parametrize("norm", ["ln", "rms"])
@pytest.mark.parametrize("dtype", ["f32", "bf16", "f16"])
@pytest.mark.parametrize("H", NORM_H)
def test_norm_parity(norm, dtype, H):
    R = 1 if H >= 11008 else (197 if H <= 1024 else 33)
    eps = 1e-6
    x = synth.norm_input(R, H, dtype)
    dy = synth.grad_input(R, H, dtype, stream=synth.S_NORM_DY)
    nf, nb, _, _ = NORM[norm]
    y, rstd = nf(x.to(DEV), eps)
    torch.cuda.synchronize()
    y_ref, r_ref = check_norm_fwd(norm, dtype, x, eps, y, rstd)
    # backward on oracle-derived inputs: y_ref rounded to T, rstd_ref to fp32
    y_in = synth.from_numpy_storage(oracle.round_to(y_ref, dtype), dtype)
    r_in = torch.from_numpy(r_ref.astype(np.float32))
    dx = nb(dy.to(DEV), y_in.to(DEV), r_in.to(DEV))
    torch.cuda.synchronize()
    check_norm_bwd(norm, dtype, dy, dec(y_in, dtype), r_in.numpy().astype(np.float64), dx)


@pytest.mark.parametrize("norm", ["ln", "rms"])
@pytest.mark.parametrize("dtype", ["f32", "bf16"])
def test_norm_coverage_rows(norm, dtype):
    """Constant row, large offset, one-hot spike, all-zero row; eps sweep."""
    H = 768
    rows = [np.full(H, 0.1), 1e3 + np.random.default_rng(0).normal(size=H), np.eye(1, H, 5)[0] * 7,
            np.zeros(H), np.random.default_rng(1).normal(size=H)]
    x = torch.tensor(np.stack(rows), dtype=torch.float32).to(DT[dtype])
    dy = synth.grad_input(len(rows), H, dtype)
    nf, nb, _, _ = NORM[norm]
    for eps in (1e-3, 1e-5, 1e-6, 1e-8):
        y, rstd = nf(x.to(DEV), eps)
        torch.cuda.synchronize()
        y_ref, r_ref = check_norm_fwd(norm, dtype, x, eps, y, rstd)
        y_in = synth.from_numpy_storage(oracle.round_to(y_ref, dtype), dtype)
        r_in = torch.from_numpy(r_ref.astype(np.float32))
        dx = nb(dy.to(DEV), y_in.to(DEV), r_in.to(DEV))
        torch.cuda.synchronize()
        check_norm_bwd(norm, dtype, dy, dec(y_in, dtype), r_in.numpy().astype(np.float64), dx)


@pytest.mark.parametrize("norm", ["ln", "rms"])
def test_norm_misaligned_inplace_deterministic(norm):
    R, H = 64, 768
    nf, nb, _, _ = NORM[norm]
    x = synth.norm_input(R, H, "bf16").to(DEV)
    dy = synth.grad_input(R, H, "bf16").to(DEV)
    y0, r0 = nf(x, 1e-6)
    y1, r1 = nf(x, 1e-6)
    dx0 = nb(dy, y0, r0)
    dx1 = nb(dy, y0, r0)
    buf = torch.empty(R * H + 1, dtype=x.dtype, device=DEV)
    xm = buf[1:].view(R, H)
    xm.copy_(x)
    ym, rm = nf(xm, 1e-6)                     # scalar path: within tolerance, not bitwise
    xi = x.clone()
    nf(xi, 1e-6, y=xi)
    torch.cuda.synchronize()
    assert torch.equal(y0.view(torch.int16), y1.view(torch.int16)) and torch.equal(r0, r1)
    assert torch.equal(dx0.view(torch.int16), dx1.view(torch.int16))
    assert torch.equal(xi.view(torch.int16), y0.view(torch.int16))
    check_norm_fwd(norm, "bf16", x.cpu(), 1e-6, ym, rm)


# ---------------------------------------------------------------------------
# full BASELINE.json sizes, sampled rows (launch configuration bench.py times)
# ---------------------------------------------------------------------------
def sample_rows(R, k=48, seed=0):
    rng = np.random.default_rng(seed)
    return sorted(set([0, 1, R - 1] + list(rng.choice(R, size=min(k, R), replace=False))))


@pytest.mark.parametrize("mode", ["bench", "coverage"])
@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4", "c5"])
def test_full_size_sampled(cfg, mode):
    """Full BASELINE sizes in bench.py's launch configuration; rows sampled
    over the whole tensor, so tiles taken over by cluster-launch-control work
    stealing are among them.  Coverage-mode inputs (10 % U(-12, 12)) put all
    four segments -- SiLU's outer ones sit at +-6.3 -- on those tiles."""
    c = synth.CONFIGS[cfg]
    R, F, H, dtype = c["R"], c["F"], c["H"], c["dtype"]
    fwd, bwd = ACT[c["act"]]
    nf, nb, of, ob = NORM[c["norm"]]
    x = synth.act_input(R, F, dtype, device=DEV, mode=mode)
    dy = synth.grad_input(R, F, dtype, device=DEV)
    y, codes = fwd(x)
    dx = bwd(dy, codes)
    xn = synth.norm_input(R, H, dtype, device=DEV)
    gn = synth.grad_input(R, H, dtype, device=DEV, stream=synth.S_NORM_DY)
    yn, rstd = nf(xn, 1e-6)
    ys = synth.norm_input(R, H, dtype, device=DEV, stream=synth.S_NORM_Y)     # bwd-only inputs
    rs = synth.rstd_input(R, device=DEV)
    dxn = nb(gn, ys, rs)
    dxc = nb(gn, yn, rstd)                  # chained fwd -> bwd
    torch.cuda.synchronize()
    rows = sample_rows(R)
    idx = torch.tensor(rows, device=DEV)
    # activation: rows are contiguous runs of F elements and F % 4 == 0
    assert F % 4 == 0
    cb = codes.view(R, F // 4)[idx].cpu()
    x_s, dy_s = x[idx].cpu(), dy[idx].cpu()
    c_ref = check_act_fwd(c["act"], dtype, x_s, y[idx], cb.reshape(-1))
    check_act_bwd(c["act"], dtype, c_ref, dy_s, dx[idx])
    if mode == "coverage":
        seg = np.bincount(((c_ref[:, None] >> np.array([0, 2, 4, 6], dtype=np.uint8)) & 3).ravel(), minlength=4)
        assert (seg > 0).all(), f"not every segment sampled: {seg}"
    # norm forward, backward on synthetic (y, rstd), chain fwd->bwd
    y_ref, r_ref = check_norm_fwd(c["norm"], dtype, xn[idx].cpu(), 1e-6, yn[idx], rstd[idx])
    check_norm_bwd(c["norm"], dtype, gn[idx].cpu(), dec(ys[idx].cpu(), dtype),
                   rs[idx].cpu().numpy().astype(np.float64), dxn[idx])
    check_norm_bwd(c["norm"], dtype, gn[idx].cpu(), y_ref, r_ref, dxc[idx])


# ---------------------------------------------------------------------------
# modules + saved bytes (a7)
# ---------------------------------------------------------------------------
def test_modules_autograd_and_saved_bytes():
    R, F, H = 128, 3072, 768
    x = synth.act_input(R, F, "bf16").to(DEV).requires_grad_(True)
    m = P.ReGELU2()
    nbytes = P.saved_bytes(m, x)
    assert nbytes == oracle.codes_bytes(R * F)                           # 8x less than bf16 x
    y = m(x)
    g = synth.grad_input(R, F, "bf16").to(DEV)
    y.backward(g)
    _, c = P.regelu2_fwd(x.detach())
    assert torch.equal(x.grad.view(torch.int16), P.regelu2_bwd(g, c).view(torch.int16))
    # MS-LN followed by a linear that saves its input: y is stored once
    xn = synth.norm_input(R, H, "bf16").to(DEV).requires_grad_(True)
    ln = P.MSLayerNorm(H)
    lin = torch.nn.Linear(H, 64, bias=False, dtype=torch.bfloat16, device=DEV)
    both = P.saved_bytes(lambda t: lin(ln(t)), xn)
    assert both == R * H * 2 + 4 * R + H * 64 * 2                        # y + rstd + weight
    exact = P.saved_bytes(lambda t: lin(torch.nn.functional.layer_norm(t, (H,))), xn)
    assert exact > both


# ---------------------------------------------------------------------------
# CUDA graphs: every entry point is capturable (no allocation, no sync, no
# host-side state) and a replayed step is bitwise identical to eager.
# ---------------------------------------------------------------------------
def test_cuda_graph_capture_replay():
    R, F, H = 256, 11008, 4096
    x = synth.act_input(R, F, "bf16").to(DEV)
    dy = synth.grad_input(R, F, "bf16").to(DEV)
    xn = synth.norm_input(R, H, "bf16").to(DEV)
    gn = synth.grad_input(R, H, "bf16").to(DEV)
    bufs = dict(y=torch.empty_like(x), dx=torch.empty_like(x), codes=torch.empty(P.codes_bytes(R * F), dtype=torch.uint8, device=DEV),
                yn=torch.empty_like(xn), dxn=torch.empty_like(xn), rstd=torch.empty(R, device=DEV))

    def step(s):
        P.msrms_fwd(xn, 1e-6, y=bufs["yn"], rstd=bufs["rstd"], stream=s)
        P.resilu2_fwd(x, y=bufs["y"], codes=bufs["codes"], stream=s)
        P.resilu2_bwd(dy, bufs["codes"], dx=bufs["dx"], stream=s)
        P.msrms_bwd(gn, bufs["yn"], bufs["rstd"], dx=bufs["dxn"], stream=s)

    s = torch.cuda.Stream()
    with torch.cuda.stream(s):
        step(s)                                   # warm-up (attributes, occupancy caches)
    s.synchronize()
    eager = {k: v.clone() for k, v in bufs.items()}
    for v in bufs.values():
        v.zero_()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        step(s)
    for v in bufs.values():
        v.zero_()
    g.replay()
    g.replay()
    torch.cuda.synchronize()
    for k in bufs:
        assert st(bufs[k]).tobytes() == st(eager[k]).tobytes(), k


def test_random_shapes():
    rng = np.random.default_rng(2406)
    for _ in range(24):
        dtype = rng.choice(["f32", "bf16", "f16"])
        kind = rng.choice(["gelu", "silu"])
        R, F = int(rng.integers(1, 40)), int(rng.integers(1, 9000))
        x = synth.act_input(R, F, dtype, mode="coverage", base=int(rng.integers(1 << 30)))
        dy = synth.grad_input(R, F, dtype)
        fwd, bwd = ACT[kind]
        y, codes = fwd(x.to(DEV))
        torch.cuda.synchronize()
        c_ref = check_act_fwd(kind, dtype, x, y, codes)
        dx = bwd(dy.to(DEV), torch.from_numpy(c_ref).to(DEV))
        torch.cuda.synchronize()
        check_act_bwd(kind, dtype, c_ref, dy, dx)
        norm = rng.choice(["ln", "rms"])
        H = int(rng.integers(1, 9000))
        xn = synth.norm_input(R, H, dtype)
        yn, r = NORM[norm][0](xn.to(DEV), 1e-6)
        torch.cuda.synchronize()
        check_norm_fwd(norm, dtype, xn, 1e-6, yn, r)


def test_more_than_2_31_elements():
    """int64 indexing end to end: an activation tensor of 2^31 + 98304
    elements (bf16, 4.3 GB), sampled rows checked against the oracle, codes
    of the last rows included."""
    R, F = (1 << 16) + 3, 32768
    x = synth.act_input(R, F, "bf16", device=DEV)
    dy = synth.grad_input(R, F, "bf16", device=DEV)
    y, codes = P.resilu2_fwd(x)
    dx = P.resilu2_bwd(dy, codes)
    torch.cuda.synchronize()
    rows = [0, 1, 40000, R - 2, R - 1]
    idx = torch.tensor(rows, device=DEV)
    c_ref = check_act_fwd("silu", "bf16", x[idx].cpu(), y[idx], codes.view(R, F // 4)[idx].reshape(-1))
    check_act_bwd("silu", "bf16", c_ref, dy[idx].cpu(), dx[idx])
    del x, dy, y, dx, codes
    torch.cuda.empty_cache()
