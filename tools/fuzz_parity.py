"""Randomised parity fuzzing (GPU): for a wall-clock budget, draw random
cases -- kernel family, dtype, shape (ragged, tiny, tile-straddling), memory
offset (16-byte aligned or not), input mode (bench / coverage / specials
spliced in), k and random sorted tables for the k-bit kernels -- run them
through the C ABI and check each against the float64 oracle with the same
bars as tests/ (DESIGN 7).  Prints one JSON summary (cases per family,
failures with their seeds).  Test infrastructure: imports oracle/ via the
tests' checkers.

    python tools/fuzz_parity.py --seconds 600 --seed 1
"""
import argparse
import json
import os
import sys
import time
import traceback

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2406_16282_b200 as P  # noqa: E402
from test_gpu_parity import (ACT, ATOL, DEV, NORM, RTOL, bits, check_act_bwd, check_act_fwd,  # noqa: E402
                             check_norm_bwd, check_norm_fwd, dec, st, ulp_dist)

DT = {"f32": torch.float32, "bf16": torch.bfloat16, "f16": torch.float16}
SPECIALS = [0.0, -0.0, 1e-30, -1e-30, 88.0, -88.0, -90.0, 100.0, -100.0, 6.3, -6.32, 3.19, -3.18, 1e4, -1e4]


def shape(rng):
    r = rng.random()
    if r < 0.05:                                # many tiles: cluster-launch-control stealing engaged
        return int(rng.integers(256, 2048)), int(rng.integers(2048, 11008))
    if r < 0.3:
        return int(rng.integers(1, 8)), int(rng.integers(1, 70))
    if r < 0.8:
        return int(rng.integers(1, 64)), int(rng.integers(1, 6000))
    return int(rng.integers(1, 4)), int(rng.integers(8000, 70000))


def act_input(rng, R, F, dtype):
    x = synth.act_input(R, F, dtype, mode="coverage" if rng.random() < 0.7 else "bench",
                        base=int(rng.integers(1 << 30)))
    if rng.random() < 0.3:                      # splice special values in at random places
        flat = x.view(-1)
        k = min(flat.numel(), 8)
        pos = torch.from_numpy(rng.choice(flat.numel(), size=k, replace=False))
        flat[pos] = torch.tensor(rng.choice(SPECIALS, size=k), dtype=torch.float32).to(x.dtype)
    return x


def placed(t, rng):
    """The tensor on the GPU, at a 16-byte aligned address or (sometimes) an
    element offset that breaks the alignment (the scalar paths)."""
    if rng.random() < 0.8:
        return t.to(DEV)
    off = int(rng.integers(1, 8))
    buf = torch.empty(t.numel() + off, dtype=t.dtype, device=DEV)
    v = buf[off:].view(t.shape)
    v.copy_(t.to(DEV))
    return v


def case_act(rng):
    dtype = str(rng.choice(["f32", "bf16", "f16"]))
    kind = str(rng.choice(["gelu", "silu"]))
    R, F = shape(rng)
    x = act_input(rng, R, F, dtype)
    dy = synth.grad_input(R, F, dtype, base=int(rng.integers(1 << 30)))
    fwd, bwd = ACT[kind]
    y, codes = fwd(placed(x, rng))
    torch.cuda.synchronize()
    c_ref = check_act_fwd(kind, dtype, x, y, codes)
    dx = bwd(placed(dy, rng), torch.from_numpy(c_ref).to(DEV))
    torch.cuda.synchronize()
    check_act_bwd(kind, dtype, c_ref, dy, dx)


def case_norm(rng):
    dtype = str(rng.choice(["f32", "bf16", "f16"]))
    norm = str(rng.choice(["ln", "rms"]))
    R, H = shape(rng)
    eps = float(rng.choice([1e-3, 1e-5, 1e-6, 1e-8]))
    x = synth.norm_input(R, H, dtype, base=int(rng.integers(1 << 30)))
    dy = synth.grad_input(R, H, dtype, base=int(rng.integers(1 << 30)))
    nf, nb, _, _ = NORM[norm]
    y, rstd = nf(placed(x, rng), eps)
    torch.cuda.synchronize()
    y_ref, r_ref = check_norm_fwd(norm, dtype, x, eps, y, rstd)
    y_in = synth.from_numpy_storage(oracle.round_to(y_ref, dtype), dtype).reshape(R, H)
    r_in = torch.from_numpy(r_ref.astype(np.float32))
    dx = nb(placed(dy, rng), placed(y_in, rng), r_in.to(DEV))
    torch.cuda.synchronize()
    check_norm_bwd(norm, dtype, dy, dec(y_in, dtype), r_in.numpy().astype(np.float64), dx)


def case_kbit(rng):
    dtype = str(rng.choice(["f32", "bf16", "f16"]))
    act = str(rng.choice(["gelu", "silu"]))
    k = int(rng.integers(1, 5))
    m = (1 << k) - 1
    thr = np.sort(rng.normal(size=m) * float(rng.choice([0.5, 3.0, 8.0])))
    if len(np.unique(thr)) < m:
        return
    lv = (rng.normal(size=m + 1)).tolist()
    R, F = shape(rng)
    x = act_input(rng, R, F, dtype)
    dy = synth.grad_input(R, F, dtype, base=int(rng.integers(1 << 30)))
    y, codes = P.stepact_fwd(placed(x, rng), act, k, thr.tolist())
    torch.cuda.synchronize()
    x64 = dec(x, dtype)
    y_ref, c_ref = oracle.stepact_fwd(act, k, thr.tolist(), x64)
    assert np.array_equal(codes.cpu().numpy(), c_ref), "k-bit codes"
    fin = np.isfinite(x64).reshape(-1)
    yr = y_ref.reshape(-1)[fin]
    assert np.all(np.abs(dec(y, dtype).reshape(-1)[fin] - yr) <= RTOL[dtype] * np.abs(yr) + ATOL[dtype]), "k-bit y"
    if dtype != "f32":
        assert ulp_dist(st(y).reshape(-1)[fin], oracle.round_to(yr, dtype), dtype).max() <= 1, "k-bit y ulp"
    dx = P.stepact_bwd(placed(dy, rng), codes, k, lv)
    torch.cuda.synchronize()
    want = oracle.stepact_bwd_contract(k, lv, c_ref, st(dy), dtype)
    assert np.array_equal(bits(st(dx)), bits(want)), "k-bit dx"


def case_swiglu(rng):
    from test_gpu_swiglu import run_case
    dtype = str(rng.choice(["f32", "bf16", "f16"]))
    R, F = shape(rng)
    g = act_input(rng, R, F, dtype)
    if not torch.isfinite(g.float()).all():
        g = torch.nan_to_num(g.float(), nan=0.0, posinf=10.0, neginf=-10.0).to(g.dtype)
    run_case(R, F, dtype, gate=g)


def case_mixed(rng):
    """Mixed-precision MS norms: fp32 x -> 16-bit y; 16-bit (dy, y) -> fp32 dx."""
    out = str(rng.choice(["bf16", "f16"]))
    norm = str(rng.choice(["ln", "rms"]))
    R, H = shape(rng)
    x = synth.norm_input(R, H, "f32", base=int(rng.integers(1 << 30)))
    dy = synth.grad_input(R, H, out, base=int(rng.integers(1 << 30)))
    nf = P.msln_fwd_mixed if norm == "ln" else P.msrms_fwd_mixed
    nb = P.msln_bwd_mixed if norm == "ln" else P.msrms_bwd_mixed
    of, ob = (oracle.msln_fwd, oracle.msln_bwd) if norm == "ln" else (oracle.msrms_fwd, oracle.msrms_bwd)
    y, rstd = nf(placed(x, rng), 1e-6, DT[out])
    torch.cuda.synchronize()
    x64 = x.double().numpy()
    y_ref, r_ref = of(x64, float(np.float32(1e-6)))
    r = rstd.cpu().numpy().astype(np.float64)
    assert np.all(np.abs(r - r_ref) <= RTOL["f32"] * 4 * r_ref), "mixed rstd"
    mu = np.abs(x64).mean(1, keepdims=True) if norm == "ln" else 0.0
    yg = dec(y, out)
    assert not (np.abs(yg - y_ref) > RTOL[out] * (np.abs(y_ref) + r_ref[:, None] * mu) + ATOL[out]).any(), "mixed y"
    dx = nb(placed(dy, rng), y, rstd)
    torch.cuda.synchronize()
    dy64 = dec(dy, out)
    ref = ob(dy64, yg, r)
    m1 = np.abs(dy64.mean(1, keepdims=True)) if norm == "ln" else 0.0
    scale = r[:, None] * (np.abs(dy64) + m1 + np.abs(yg) * np.abs(dy64 * yg).mean(1, keepdims=True))
    assert not (np.abs(dx.cpu().numpy().astype(np.float64) - ref) > RTOL["f32"] * 4 * scale + ATOL["f32"]).any(), "mixed dx"


FAMILIES = {"act": case_act, "norm": case_norm, "kbit": case_kbit, "swiglu": case_swiglu, "mixed": case_mixed}


def run_cases(seed: int, n: int):
    """n cases from seed (the pytest entry point); returns the failures."""
    fails = []
    for i in range(n):
        s = seed * 1_000_003 + i
        rng = np.random.default_rng(s)
        fam = str(rng.choice(list(FAMILIES)))
        try:
            FAMILIES[fam](rng)
        except Exception as e:
            fails.append((fam, s, repr(e)[:300]))
    return fails


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--seconds", type=float, default=300)
    ap.add_argument("--seed", type=int, default=1)
    a = ap.parse_args()
    t0 = time.time()
    counts = {k: 0 for k in FAMILIES}
    fails = []
    i = 0
    while time.time() - t0 < a.seconds:
        seed = a.seed * 1_000_003 + i
        rng = np.random.default_rng(seed)
        fam = str(rng.choice(list(FAMILIES)))
        try:
            FAMILIES[fam](rng)
            counts[fam] += 1
        except Exception as e:  # record and continue
            fails.append({"family": fam, "seed": seed, "error": repr(e)[:300],
                          "where": traceback.format_exc().splitlines()[-3][:200]})
        i += 1
    print(json.dumps({"cases": i, "per_family": counts, "failures": len(fails), "first_failures": fails[:20],
                      "seconds": round(time.time() - t0, 1), "seed": a.seed}))


if __name__ == "__main__":
    main()
