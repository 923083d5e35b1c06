"""Debug aid: where do the TMA-pipeline and simple-kernel stepact paths differ?"""
import sys, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..")); sys.path.insert(0, os.path.join(os.path.dirname(__file__), "..", "tests"))
import numpy as np, torch
import synth, oracle
import paper_2406_16282_b200 as P
from test_gpu_parity import st
DEV = "cuda"
for k in (1, 2, 4):
    for dtype in ("f32", "bf16"):
        rng = np.random.default_rng(10 + k)
        if k == 1: c, s = [0.0], [0.0, 1.0]
        elif k == 2:
            c, s = oracle.regelu2d_table(); c, s = list(c), list(s)
        else:
            c = sorted(rng.normal(size=15) * 3); s = list(rng.normal(size=16))
        R, F = 33, 4099
        x = synth.act_input(R, F, dtype, mode="coverage").to(DEV)
        y0, c0 = P.stepact_fwd(x, "silu", k, c)
        cb = torch.empty(c0.numel() + 1, dtype=torch.uint8, device=DEV)
        y1, c1 = P.stepact_fwd(x, "silu", k, c, codes=cb[1:])
        torch.cuda.synchronize()
        a = st(y0).reshape(-1).view(np.uint16 if dtype == "bf16" else np.uint32)
        b = st(y1).reshape(-1).view(np.uint16 if dtype == "bf16" else np.uint32)
        xs = st(x).reshape(-1).view(np.uint16 if dtype == "bf16" else np.uint32)
        bad = np.nonzero(a != b)[0]
        print(k, dtype, "codes equal", torch.equal(c0, c1), "y mismatches", len(bad))
        for i in bad[:8]:
            print("   i", i, "x bits %x" % xs[i], "x", x.reshape(-1)[i].item(), "tma %x" % a[i], "simple %x" % b[i])
