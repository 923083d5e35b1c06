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
        for k, thr, lv in ((1, [0.0], [0.0, 1.0]), (2, tables.REGELU2["c"], tables.levels(tables.REGELU2))):
            y, c = P.stepact_fwd(x, "gelu", k, thr)
            P.stepact_bwd(dy, c, k, lv)
    for (R, H) in ((3, 7), (33, 768), (9, 4096), (5, 5120), (2, 40000)):
        xn = synth.norm_input(R, H, dt).to(dev)
        gn = synth.grad_input(R, H, dt).to(dev)
        for fwd, bwd in ((P.msln_fwd, P.msln_bwd), (P.msrms_fwd, P.msrms_bwd)):
            yn, r = fwd(xn, 1e-6)
            bwd(gn, yn, r)
torch.cuda.synchronize()
print("sanitize driver ok")
