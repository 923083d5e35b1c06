"""Fixed vs per-byte cost of the activation kernels across library variants
(tools/sweep.py's variant syntax: name:DEF1,DEF2 or name:@path/to/lib.so):
time act_fwd / act_bwd of each variant and a torch copy at several row counts
of one width with the bench protocol (L2 flushed by a 2 x L2 read, CUDA
events, median of --iters), fit t = a + bytes / r per (variant, kernel).
Prints one JSON line per point and one per fit."""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tools"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2406_16282_b200 import build as B  # noqa: E402
from sweep import load  # noqa: E402

DT = {"f32": 0, "bf16": 1, "f16": 2}
THR4 = (ctypes.c_double * 15)(*[-3.0 + 0.4 * i for i in range(15)])   # as tools/sweep.py
THR3 = (ctypes.c_double * 7)(*[-3.0 + 1.0 * i for i in range(7)])


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--act", default="silu")
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--cols", type=int, default=11008)
    ap.add_argument("--rows", default="1024,2048,4096,8192,16384")
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--kernels", default="fwd,bwd")
    ap.add_argument("--variants", nargs="+", default=["base:"])
    ap.add_argument("--build-only", action="store_true")
    ap.add_argument("--norm", default="rms", help="ln | rms, for the norm kernels (cols = H)")
    a = ap.parse_args()
    libs = {}
    for v in a.variants:
        name, _, defs = v.partition(":")
        libs[name] = (os.path.join(ROOT, defs[1:]) if defs.startswith("@") else
                      B.build_variant(name, [d for d in defs.split(",") if d],
                                      sources=[s for s in B.SOURCES if s != "fit.cu"]))
    if a.build_only:
        return
    dev = torch.device("cuda")
    l2 = torch.cuda.get_device_properties(dev).L2_cache_size
    flush = torch.ones(max(2 * l2, 256 << 20) // 4, device=dev)
    sink = torch.zeros((), device=dev)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    act = "regelu2" if a.act == "gelu" else "resilu2"
    L = {k: load(p) for k, p in libs.items()}
    pts = {}
    for R in [int(r) for r in a.rows.split(",")]:
        x = synth.act_input(R, a.cols, a.dtype, device=dev)
        dy = synth.grad_input(R, a.cols, a.dtype, device=dev)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        n, b = x.numel(), x.element_size()
        codes = torch.empty((n + 3) // 4, dtype=torch.uint8, device=dev)
        nb = 2 * b * n + (n + 3) // 4
        codes4 = torch.empty((n + 1) // 2, dtype=torch.uint8, device=dev)
        rstd = torch.rand(R, device=dev) + 0.5
        if "nbwd" in a.kernels or "swb" in a.kernels:
            x2, y2 = torch.empty_like(x), torch.empty_like(x)
        if "nbwd" in a.kernels:
            y.copy_(synth.norm_input(R, a.cols, a.dtype, device=dev))
        codes3 = torch.empty((3 * n + 7) // 8, dtype=torch.uint8, device=dev)
        ak = 0 if a.act == "gelu" else 1
        fns = {("torch", "copy"): (lambda: (y.copy_(x), 0)[1], 2 * b * n)}
        for name, lib in L.items():
            f, bw = getattr(lib, act + "_fwd"), getattr(lib, act + "_bwd")
            if "fwd" in a.kernels:
                fns[(name, "fwd")] = (lambda f=f: f(x.data_ptr(), y.data_ptr(), codes.data_ptr(), R, a.cols,
                                                    DT[a.dtype], sp), nb)
            nrm = "msln" if a.norm == "ln" else "msrms"
            if "nfwd" in a.kernels:
                nf = getattr(lib, nrm + "_fwd")
                fns[(name, "nfwd")] = (lambda nf=nf: nf(x.data_ptr(), y.data_ptr(), rstd.data_ptr(), R, a.cols, 1e-6,
                                                        DT[a.dtype], sp), 2 * b * n + 4 * R)
            if "nbwd" in a.kernels:
                nbk = getattr(lib, nrm + "_bwd")
                fns[(name, "nbwd")] = (lambda nbk=nbk: nbk(dy.data_ptr(), y.data_ptr(), rstd.data_ptr(), dx.data_ptr(), R,
                                                           a.cols, DT[a.dtype], sp), 3 * b * n + 4 * R)
            if "swf" in a.kernels:
                fns[(name, "swf")] = (lambda lib=lib: lib.reswiglu2_fwd(x.data_ptr(), dy.data_ptr(), y.data_ptr(),
                                                                        dx.data_ptr(), codes.data_ptr(), R, a.cols,
                                                                        DT[a.dtype], sp), 4 * b * n + (n + 3) // 4)
            if "swb" in a.kernels:
                fns[(name, "swb")] = (lambda lib=lib: lib.reswiglu2_bwd(y.data_ptr(), dy.data_ptr(), dx.data_ptr(),
                                                                        codes.data_ptr(), x2.data_ptr(), y2.data_ptr(),
                                                                        R, a.cols, DT[a.dtype], sp), 5 * b * n + (n + 3) // 4)
            if "step4" in a.kernels:
                fns[(name, "step4")] = (lambda lib=lib: lib.stepact_fwd(ak, 4, ctypes.addressof(THR4), x.data_ptr(),
                                                                      y.data_ptr(), codes4.data_ptr(), R, a.cols,
                                                                      DT[a.dtype], sp), 2 * b * n + (n + 1) // 2)
            if "step3" in a.kernels:
                fns[(name, "step3")] = (lambda lib=lib: lib.stepact_fwd(ak, 3, ctypes.addressof(THR3), x.data_ptr(),
                                                                      y.data_ptr(), codes3.data_ptr(), R, a.cols,
                                                                      DT[a.dtype], sp), 2 * b * n + (3 * n + 7) // 8)
            if "bwd" in a.kernels:
                fns[(name, "bwd")] = (lambda bw=bw: bw(dy.data_ptr(), codes.data_ptr(), dx.data_ptr(), R, a.cols,
                                                       DT[a.dtype], sp), nb)
        for key, (fn, nbytes) in fns.items():
            for _ in range(3):
                assert fn() == 0
            ev = []
            for _ in range(a.iters):
                sink.copy_(flush.sum())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                fn()
                e1.record(st)
                ev.append((e0, e1))
            torch.cuda.synchronize()
            us = float(np.median([e0.elapsed_time(e1) * 1e3 for e0, e1 in ev]))
            pts.setdefault(key, []).append((nbytes, us))
            print(json.dumps({"variant": key[0], "kernel": key[1], "rows": R, "cols": a.cols, "bytes": nbytes,
                              "us": round(us, 2), "GB/s": round(nbytes / us / 1e3, 1)}), flush=True)
        del x, dy, y, dx, codes
        torch.cuda.empty_cache()
    for key, v in pts.items():
        Bv = np.array([p[0] for p in v], dtype=np.float64)
        T = np.array([p[1] for p in v])
        A = np.stack([np.ones_like(Bv), Bv], 1)
        (c0, c1), *_ = np.linalg.lstsq(A, T, rcond=None)
        print(json.dumps({"fit": key[1], "variant": key[0], "fixed_us": round(float(c0), 2),
                          "GB/s_marginal": round(1e-3 / float(c1), 1)}))


if __name__ == "__main__":
    main()
