"""Run every C-ABI entry point once on small, ragged shapes (for
compute-sanitizer memcheck / racecheck / synccheck / initcheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2406_16282_b200 as P  # noqa: E402
from paper_2406_16282_b200 import tables  # noqa: E402

dev = "cuda"
for dt in ("f32", "bf16", "f16"):
    for (R, F) in ((3, 7), (37, 3072), (5, 40000)):
        x = synth.act_input(R, F, dt, mode="coverage").to(dev)
        dy = synth.grad_input(R, F, dt).to(dev)
        for fwd, bwd in ((P.regelu2_fwd, P.regelu2_bwd), (P.resilu2_fwd, P.resilu2_bwd)):
            y, c = fwd(x)
            bwd(dy, c)
        h, a, c = P.reswiglu2_fwd(x, dy)
        P.reswiglu2_bwd(dy, dy, a, c)
        for k, thr, lv in ((1, [0.0], [0.0, 1.0]), (2, tables.REGELU2["c"], tables.levels(tables.REGELU2)),
                           (3, [-3.0 + 1.0 * i for i in range(7)], [i / 7 for i in range(8)]),
                           (4, [-3.0 + 0.4 * i for i in range(15)], [i / 15 for i in range(16)])):
            for act in ("gelu", "silu"):            # GELU 16-bit: y table; SiLU 16-bit k >= 3: code table
                y, c = P.stepact_fwd(x, act, k, thr)
                P.stepact_bwd(dy, c, k, lv)
            cb = torch.empty(c.numel() + 1, dtype=torch.uint8, device=dev)   # misaligned codes: simple kernels
            y, c = P.stepact_fwd(x, "silu", k, thr, codes=cb[1:])
            P.stepact_bwd(dy, c, k, lv)
    for (R, H) in ((3, 7), (33, 768), (9, 4096), (5, 5120), (2, 40000), (2, 65537), (1, 262144)):
        xn = synth.norm_input(R, H, dt).to(dev)
        gn = synth.grad_input(R, H, dt).to(dev)
        for fwd, bwd in ((P.msln_fwd, P.msln_bwd), (P.msrms_fwd, P.msrms_bwd)):
            yn, r = fwd(xn, 1e-6)
            bwd(gn, yn, r)
        if dt != "f32":                                  # mixed: fp32 residual in, 16-bit y out
            for fwd, bwd in ((P.msln_fwd_mixed, P.msln_bwd_mixed), (P.msrms_fwd_mixed, P.msrms_bwd_mixed)):
                ym, rm = fwd(xn.float(), 1e-6, xn.dtype)
                bwd(gn, ym, rm)
# coefficient fitter (fp64): objective for k = 1..3, a short anneal + refine
for act in ("gelu", "silu"):
    for k in (1, 2, 3):
        P_ = P.ops.fit_n_params(k)
        th = torch.randn(67, P_, dtype=torch.float64, device=dev)
        P.ops.fit_objective(th, act, k=k)
        P.ops.fit_objective(th, act, k=k, objective="dh")
    best, cth, cj = P.ops.fit_anneal(act, chains=150, iters=20)
    P.ops.fit_refine(cth, act, iters=2)
    for k in (1, 2, 4):
        P.ops.fit_anneal(act, k=k, chains=70, iters=10, projected=True)
torch.cuda.synchronize()
print("sanitize driver ok")
