import sys, time, os
sys.path.insert(0, "/root/repo")
import torch
from paper_2406_16282_b200 import fit as gfit, ops
for act in ("gelu", "silu"):
    for k, chains, iters, ri in ((1, 4096, 500, 40), (2, 8192, 1500, 40), (3, 8192, 4000, 20), (4, 4096, 8000, 8)):
        torch.cuda.synchronize(); t = time.time()
        f = gfit.fit(act, k=k, chains=chains, iters=iters, refine_iters=ri)
        torch.cuda.synchronize()
        print(act, k, chains, iters, ri, "J=%.6e" % f.J, "%.2fs" % (time.time() - t), [round(c, 3) for c in f.c], flush=True)
