"""Tuning aid for the GPU coefficient fitter: J reached / J(paper) for
several annealing schedules (prints one line per setting)."""
import itertools, sys, os, time
sys.path.insert(0, os.path.join(os.path.dirname(__file__), ".."))
import torch
from paper_2406_16282_b200 import ops, fit as gfit
from bench import PAPER_THETA  # noqa: E402

for (act, obj), (chains, iters, t0) in itertools.product(list(PAPER_THETA), [
        (4096, 2000, 0.1), (4096, 4000, 0.1), (16384, 2000, 0.1), (56832, 1000, 0.1), (56832, 3000, 0.1),
        (4096, 2000, 1.0)]):
    Jp = float(gfit.objective(PAPER_THETA[(act, obj)], act, objective=obj)[0])
    for seed in (7, 8):
        t = time.time()
        f = gfit.fit(act, objective=obj, chains=chains, iters=iters, t0=t0, seed=seed)
        print(act, obj, chains, iters, t0, seed, "ratio %.7f" % (f.J / Jp), "%.2fs" % (time.time() - t),
              [round(v, 5) for v in f.a + f.c], flush=True)
