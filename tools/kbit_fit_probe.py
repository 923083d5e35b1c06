"""k = 1..4 GPU fits of GELU / SiLU (Eq. 15): plain annealing of all
parameters vs variable projection (thresholds annealed, weights by least
squares), each followed by the LM refinement.  Prints J and time."""
import sys, time, os
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2406_16282_b200 import fit as gfit
for act in ("gelu", "silu"):
    for k, chains, iters, ri in ((1, 4096, 500, 40), (2, 8192, 1500, 40), (3, 8192, 4000, 20), (4, 4096, 8000, 8)):
        for proj in (False, True):
            torch.cuda.synchronize(); t = time.time()
            f = gfit.fit(act, k=k, chains=chains, iters=iters if not proj else iters // 2 + 100, refine_iters=ri,
                         projected=proj)
            torch.cuda.synchronize()
            print(act, k, "vp" if proj else "sa", chains, iters, ri, "J=%.6e" % f.J, "%.2fs" % (time.time() - t),
                  [round(c, 3) for c in f.c], flush=True)
