"""ncu driver: one k = 4 step-activation forward and backward (SiLU, C4
shape, bf16) through the binding, nothing else on the GPU except the input
generation.  ncu --set full -k regex:ew_tma -c 2 python tools/step4_prof_driver.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2406_16282_b200 as P  # noqa: E402
import synth  # noqa: E402

cfg = synth.CONFIGS["c4"]
x = synth.act_input(cfg["R"], cfg["F"], cfg["dtype"], device=torch.device("cuda"))
dy = synth.grad_input(cfg["R"], cfg["F"], cfg["dtype"], device=torch.device("cuda"))
thr = [-3.0 + 0.4 * i for i in range(15)]
lv = [i / 15 for i in range(16)]
y, codes = P.stepact_fwd(x, "silu", 4, thr)
dx = P.stepact_bwd(dy, codes, 4, lv)
torch.cuda.synchronize()
print("step4 driver ok", codes.numel())
