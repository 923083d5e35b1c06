"""Tuning sweep: time one kernel of several liblmbp variants (built with
different -D parameters by paper_2406_16282_b200.build.build_variant) on a
BASELINE config shape, L2 flushed (read of 2 x L2) before every launch, CUDA
events on the launching stream.  Prints one JSON line per (variant, kernel).

    python tools/sweep.py --config c4 --variants base:  s3:LMBP_TMA_STAGES=3 ...
"""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import synth  # noqa: E402
from paper_2406_16282_b200 import build as B  # noqa: E402
from paper_2406_16282_b200._lib import SIGNATURES  # noqa: E402

DT = {"f32": 0, "bf16": 1, "f16": 2}


def load(path):
    L = ctypes.CDLL(path)
    for name, (res, args) in SIGNATURES.items():
        f = getattr(L, name, None)          # sweep variants are built without the fitter
        if f is not None:
            f.restype, f.argtypes = res, args
    return L


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c4")
    ap.add_argument("--variants", nargs="+", default=["base:"])
    ap.add_argument("--iters", type=int, default=30)
    ap.add_argument("--kernels", default="act_fwd,act_bwd,norm_fwd,norm_bwd")
    ap.add_argument("--build-only", action="store_true")
    ap.add_argument("--sources", default=None, help="comma list of .cu files compiled with the variant's -D set "
                                                     "(the rest are linked from the product build)")
    ap.add_argument("--yoff", type=int, default=0, help="offset y by this many bytes (address-interaction probe)")
    a = ap.parse_args()
    libs = {}
    for v in a.variants:
        name, _, defs = v.partition(":")
        if defs.startswith("@"):          # a prebuilt library, e.g. from another commit
            libs[name] = os.path.join(ROOT, defs[1:])
        else:
            libs[name] = B.build_variant(name, [d for d in defs.split(",") if d],
                                         sources=(a.sources.split(",") if a.sources else
                                                  [s for s in B.SOURCES if s != "fit.cu"]))
    if a.build_only:
        return
    cfg = synth.CONFIGS[a.config]
    R, F, H, dt = cfg["R"], cfg["F"], cfg["H"], cfg["dtype"]
    dev = torch.device("cuda")
    x = synth.act_input(R, F, dt, device=dev)
    dy = synth.grad_input(R, F, dt, device=dev)
    ybuf = torch.empty(x.numel() * x.element_size() + a.yoff, dtype=torch.uint8, device=dev)
    y = ybuf[a.yoff:].view(x.dtype).view(x.shape)
    dx = torch.empty_like(dy)
    x2, y2 = torch.empty_like(dy), torch.empty_like(dy)
    codes = torch.empty((R * F + 3) // 4, dtype=torch.uint8, device=dev)
    codes4 = torch.empty((R * F + 1) // 2, dtype=torch.uint8, device=dev)
    thr2 = (ctypes.c_double * 3)(-3.1858810036855245, -0.001178821281161997, 3.190832613414926)
    lv2 = (ctypes.c_double * 4)(0.0, -0.04922261145617846, 1.0487405950855513, 1.0)
    thr4 = (ctypes.c_double * 15)(*[-3.0 + 0.4 * i for i in range(15)])
    thr3 = (ctypes.c_double * 7)(*[-3.0 + 1.0 * i for i in range(7)])
    lv3 = (ctypes.c_double * 8)(*[i / 7 for i in range(8)])
    codes3 = torch.empty((R * F * 3 + 7) // 8, dtype=torch.uint8, device=dev)
    lv4 = (ctypes.c_double * 16)(*[i / 15 for i in range(16)])
    xn = synth.norm_input(R, H, dt, device=dev)
    gn = synth.grad_input(R, H, dt, device=dev)
    yn, dxn = torch.empty_like(xn), torch.empty_like(gn)
    xn32 = xn.float()                                 # fp32 residual stream for the mixed norms
    dxn32 = torch.empty_like(xn32)
    rstd = torch.empty(R, dtype=torch.float32, device=dev)
    flush = torch.ones((2 * torch.cuda.get_device_properties(dev).L2_cache_size) // 4, device=dev)
    sink = torch.zeros((), device=dev)
    st = torch.cuda.current_stream()
    sp = st.cuda_stream
    b = synth.ELEM_BYTES[dt]
    n = R * F
    nbytes = {"ncopy": 2 * b * R * H, "copy": 2 * b * n, "act_fwd": 2 * b * n + (n + 3) // 4, "act_bwd": 2 * b * n + (n + 3) // 4,
              "norm_fwd": (2 * b * H + 4) * R, "norm_bwd": (3 * b * H + 4) * R,
              "step2_fwd": 2 * b * n + (n + 3) // 4, "step4_fwd": 2 * b * n + (n + 1) // 2,
              "step4_bwd": 2 * b * n + (n + 1) // 2, "step3_fwd": 2 * b * n + (3 * n + 7) // 8,
              "step3_bwd": 2 * b * n + (3 * n + 7) // 8,
              "mnorm_fwd": (4 * H + b * H + 4) * R, "mnorm_bwd": (2 * b * H + 4 + 4 * H) * R,
              "swiglu_fwd": 4 * b * n + (n + 3) // 4, "swiglu_bwd": 5 * b * n + (n + 3) // 4}
    act = "regelu2" if cfg["act"] == "gelu" else "resilu2"
    nrm = "msln" if cfg["norm"] == "ln" else "msrms"
    for name, path in libs.items():
        L = load(path)
        calls = {
            "copy": lambda: (y.copy_(x), 0)[1],     # torch copy of the same tensors: same-footprint reference
            "ncopy": lambda: (yn.copy_(xn), 0)[1],  # torch copy of the norm tensor
            "act_fwd": lambda: getattr(L, act + "_fwd")(x.data_ptr(), y.data_ptr(), codes.data_ptr(), R, F, DT[dt], sp),
            "act_bwd": lambda: getattr(L, act + "_bwd")(dy.data_ptr(), codes.data_ptr(), dx.data_ptr(), R, F, DT[dt], sp),
            "norm_fwd": lambda: getattr(L, nrm + "_fwd")(xn.data_ptr(), yn.data_ptr(), rstd.data_ptr(), R, H, 1e-6,
                                                         DT[dt], sp),
            "norm_bwd": lambda: getattr(L, nrm + "_bwd")(gn.data_ptr(), yn.data_ptr(), rstd.data_ptr(), dxn.data_ptr(),
                                                         R, H, DT[dt], sp),
        }
        ak = 0 if cfg["act"] == "gelu" else 1
        calls["step2_fwd"] = lambda: L.stepact_fwd(ak, 2, ctypes.addressof(thr2), x.data_ptr(), y.data_ptr(),
                                                   codes.data_ptr(), R, F, DT[dt], sp)
        calls["step4_fwd"] = lambda: L.stepact_fwd(ak, 4, ctypes.addressof(thr4), x.data_ptr(), y.data_ptr(),
                                                   codes4.data_ptr(), R, F, DT[dt], sp)
        mk = 0 if cfg["norm"] == "ln" else 1
        mfwd = getattr(L, nrm + "_fwd_mixed", None)
        mbwd = getattr(L, nrm + "_bwd_mixed", None)
        calls["mnorm_fwd"] = lambda: mfwd(xn32.data_ptr(), yn.data_ptr(), rstd.data_ptr(), R, H, 1e-6, DT[dt], sp)
        calls["mnorm_bwd"] = lambda: mbwd(gn.data_ptr(), yn.data_ptr(), rstd.data_ptr(), dxn32.data_ptr(), R, H,
                                          DT[dt], sp)
        calls["step3_fwd"] = lambda: L.stepact_fwd(ak, 3, ctypes.addressof(thr3), x.data_ptr(), y.data_ptr(),
                                                   codes3.data_ptr(), R, F, DT[dt], sp)
        calls["step3_bwd"] = lambda: L.stepact_bwd(3, ctypes.addressof(lv3), dy.data_ptr(), codes3.data_ptr(),
                                                   dx.data_ptr(), R, F, DT[dt], sp)
        calls["step4_bwd"] = lambda: L.stepact_bwd(4, ctypes.addressof(lv4), dy.data_ptr(), codes4.data_ptr(),
                                                   dx.data_ptr(), R, F, DT[dt], sp)
        # fused ReSwiGLU2 on (x as gate, dy as up): h -> y, a -> dx; bwd reads (dy as dh, dy as up, dx as a)
        calls["swiglu_fwd"] = lambda: L.reswiglu2_fwd(x.data_ptr(), dy.data_ptr(), y.data_ptr(), dx.data_ptr(),
                                                      codes.data_ptr(), R, F, DT[dt], sp)
        calls["swiglu_bwd"] = lambda: L.reswiglu2_bwd(y.data_ptr(), dy.data_ptr(), dx.data_ptr(), codes.data_ptr(),
                                                      x2.data_ptr(), y2.data_ptr(), R, F, DT[dt], sp)
        calls["act_fwd"]()
        calls["norm_fwd"]()
        calls["step4_fwd"]()
        for k in a.kernels.split(","):
            rc0 = calls[k]()
            if rc0 != 0:                      # e.g. a shape the GPU refuses (> 1024 threads)
                torch.cuda.synchronize()
                print(json.dumps({"variant": name, "config": a.config, "kernel": k, "error": rc0}), flush=True)
                continue
            for _ in range(3):
                calls[k]()
            ts = []
            for _ in range(a.iters):
                sink.copy_(flush.sum())
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                rc = calls[k]()
                e1.record(st)
                assert rc == 0, rc
                ts.append((e0, e1))
            torch.cuda.synchronize()
            us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ts)
            med = us[len(us) // 2]
            print(json.dumps({"variant": name, "config": a.config, "kernel": k, "yoff": a.yoff, "us_med": round(med, 2),
                              "us_min": round(us[0], 2), "GB/s": round(nbytes[k] / med / 1e3, 1),
                              "frac": round(nbytes[k] / med / 1e3 / 6536, 4)}), flush=True)


if __name__ == "__main__":
    main()
