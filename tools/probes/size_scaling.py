"""Fixed cost vs per-byte cost of the activation kernels: time act_fwd,
act_bwd (and a torch copy of the same bytes) at several row counts of one
width with the bench protocol (L2 flushed by a 2 x L2 read, CUDA events,
median of 30) and fit t = a + bytes / r.  Prints one JSON line per point and
one per fit."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
import paper_2406_16282_b200 as P  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--act", default="silu")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--cols", type=int, default=11008)
    ap.add_argument("--rows", default="1024,2048,4096,8192,16384,32768")
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.ones(max(2 * l2, 256 << 20) // 4, device=dev)
    sink = torch.zeros((), device=dev)
    fwd, bwd = (P.regelu2_fwd, P.regelu2_bwd) if a.act == "gelu" else (P.resilu2_fwd, P.resilu2_bwd)
    pts = {"fwd": [], "bwd": [], "copy": []}
    for R in [int(r) for r in a.rows.split(",")]:
        x = synth.act_input(R, a.cols, a.dtype, device=dev)
        dy = synth.grad_input(R, a.cols, a.dtype, device=dev)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        codes = torch.empty(P.codes_bytes(x.numel()), dtype=torch.uint8, device=dev)
        n, b = x.numel(), x.element_size()
        nb = 2 * b * n + (n + 3) // 4
        fns = {"fwd": (lambda: fwd(x, y=y, codes=codes), nb), "bwd": (lambda: bwd(dy, codes, dx=dx), nb),
               "copy": (lambda: y.copy_(x), 2 * b * n)}
        for k, (fn, nbytes) in fns.items():
            for _ in range(3):
                fn()
            ev = []
            for _ in range(a.iters):
                sink.copy_(flush.sum())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                fn()
                e1.record()
                ev.append((e0, e1))
            torch.cuda.synchronize()
            us = float(np.median([e0.elapsed_time(e1) * 1e3 for e0, e1 in ev]))
            pts[k].append((nbytes, us))
            print(json.dumps({"kernel": k, "rows": R, "cols": a.cols, "bytes": nbytes, "us": round(us, 2),
                              "GB/s": round(nbytes / us / 1e3, 1)}), flush=True)
        del x, dy, y, dx, codes
        torch.cuda.empty_cache()
    for k, v in pts.items():
        B = np.array([p[0] for p in v], dtype=np.float64)
        T = np.array([p[1] for p in v])
        A = np.stack([np.ones_like(B), B], 1)
        (c0, c1), *_ = np.linalg.lstsq(A, T, rcond=None)
        print(json.dumps({"fit": k, "fixed_us": round(float(c0), 2), "GB/s_marginal": round(1e-3 / float(c1), 1)}))


if __name__ == "__main__":
    main()
