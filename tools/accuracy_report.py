"""Accuracy report of the GPU kernels against the float64 oracle (beyond the
pass/fail bars of the tests): per kernel and dtype, the worst error relative
to its tolerance scale, and for 16-bit outputs the ulp histogram / fraction
correctly rounded.  Writes JSON to the path given (default stdout)."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
import synth  # noqa: E402
import paper_2406_16282_b200 as P  # noqa: E402
from test_gpu_parity import dec, st, ulp_dist  # noqa: E402

DEV = "cuda"
out = {}
for dtype in ("f32", "bf16", "f16"):
    for kind, fwd in (("gelu", P.regelu2_fwd), ("silu", P.resilu2_fwd)):
        x = synth.act_input(512, 11008, dtype, mode="coverage")
        y, codes = fwd(x.to(DEV))
        torch.cuda.synchronize()
        x64 = dec(x, dtype)
        y_ref, c_ref = oracle.act_fwd(kind, x64)
        fin = np.isfinite(x64).reshape(-1)
        yr = y_ref.reshape(-1)[fin]
        yg = dec(y, dtype).reshape(-1)[fin]
        big = np.abs(yr) > 1e-30
        rel = np.abs(yg - yr)[big] / np.abs(yr[big])
        rec = {"elements": int(yr.size), "codes_equal": bool(np.array_equal(codes.cpu().numpy(), c_ref)),
               "max_rel_err": float(rel.max()), "mean_rel_err": float(rel.mean())}
        if dtype != "f32":
            d = ulp_dist(st(y).reshape(-1)[fin], oracle.round_to(yr, dtype), dtype)
            rec["ulp_histogram"] = {int(k): int(v) for k, v in zip(*np.unique(d, return_counts=True))}
            rec["correctly_rounded_fraction"] = float((d == 0).mean())
        out[f"{kind}_fwd_{dtype}"] = rec
    for norm, (nf, of) in (("ln", (P.msln_fwd, oracle.msln_fwd)), ("rms", (P.msrms_fwd, oracle.msrms_fwd))):
        xn = synth.norm_input(256, 4096, dtype)
        yn, r = nf(xn.to(DEV), 1e-6)
        torch.cuda.synchronize()
        yr, rr = of(dec(xn, dtype), float(np.float32(1e-6)))
        yg = dec(yn, dtype)
        mu = np.abs(dec(xn, dtype).mean(1, keepdims=True)) if norm == "ln" else 0.0
        scale = np.abs(yr) + rr[:, None] * mu + 1e-30
        out[f"{norm}_fwd_{dtype}"] = {"max_err_over_scale": float((np.abs(yg - yr) / scale).max()),
                                      "max_rstd_rel_err": float((np.abs(r.cpu().numpy() - rr) / rr).max())}
text = json.dumps(out, indent=1)
if len(sys.argv) > 1:
    open(sys.argv[1], "w").write(text)
print(text)
