"""Driver for ncu captures of the coefficient-fitter kernels: one batched
objective launch per activation, one annealing launch, one refinement launch,
one variable-projection annealing launch."""
import os, sys
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2406_16282_b200 import ops
from bench import PAPER_THETA
g = torch.Generator(device="cuda").manual_seed(2406)
n = 148 * 3 * 128 * 4
for act in ("gelu", "silu"):
    th = torch.tensor(PAPER_THETA[(act, "h")], dtype=torch.float64, device="cuda")
    batch = (th + 0.05 * torch.randn(n, 5, dtype=torch.float64, device="cuda", generator=g)).contiguous()
    ops.fit_objective(batch, act)
best, cth, cj = ops.fit_anneal("silu", chains=148 * 3 * 128, iters=200)
ops.fit_refine(cth, "silu", iters=5)
ops.fit_anneal("silu", chains=148 * 3 * 128, iters=200, projected=True)
torch.cuda.synchronize()
print("ok")
