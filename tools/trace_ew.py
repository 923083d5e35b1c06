"""Timeline of one elementwise-pipeline launch (diagnostic LMBP_TRACE build):
per running CTA the SM, entry time, first tile's arrival, exit time and tile
count (globaltimer ns), against the CUDA-event time of the same launch.
Prints one JSON summary per (variant, config, kernel)."""
import argparse
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import synth  # noqa: E402
from paper_2406_16282_b200 import build as B  # noqa: E402

DT = {"f32": 0, "bf16": 1, "f16": 2}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--variants", nargs="+", default=["trace:LMBP_TRACE"])
    ap.add_argument("--configs", default="c2,c4")
    ap.add_argument("--build-only", action="store_true")
    a = ap.parse_args()
    libs = {}
    for v in a.variants:
        name, _, defs = v.partition(":")
        if defs.startswith("@"):
            libs[name] = os.path.join(ROOT, defs[1:])
        else:
            libs[name] = B.build_variant(name, [d for d in defs.split(",") if d],
                                         sources=[s for s in B.SOURCES if s != "fit.cu"])
    if a.build_only:
        return
    dev = torch.device("cuda")
    flush = torch.ones((2 * torch.cuda.get_device_properties(dev).L2_cache_size) // 4, device=dev)
    sink = torch.zeros((), device=dev)
    st = torch.cuda.current_stream()
    buf = (ctypes.c_ulonglong * (8192 * 5))()
    for cname in a.configs.split(","):
        cfg = synth.CONFIGS[cname]
        R, F, dt = cfg["R"], cfg["F"], cfg["dtype"]
        x = synth.act_input(R, F, dt, device=dev)
        dy = synth.grad_input(R, F, dt, device=dev)
        y, dx = torch.empty_like(x), torch.empty_like(x)
        codes = torch.empty((R * F + 3) // 4, dtype=torch.uint8, device=dev)
        act = "regelu2" if cfg["act"] == "gelu" else "resilu2"
        for name, path in libs.items():
            L = ctypes.CDLL(path)
            L.lmbp_trace_act.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_int]
            L.lmbp_trace_units_act.argtypes = [ctypes.c_void_p, ctypes.c_int]
            f = getattr(L, act + "_fwd")
            b = getattr(L, act + "_bwd")
            for fn in (f, b):
                fn.argtypes = [ctypes.c_void_p] * 3 + [ctypes.c_int64, ctypes.c_int64, ctypes.c_int, ctypes.c_void_p]
            calls = {"act_fwd": lambda: f(x.data_ptr(), y.data_ptr(), codes.data_ptr(), R, F, DT[dt], st.cuda_stream),
                     "act_bwd": lambda: b(dy.data_ptr(), codes.data_ptr(), dx.data_ptr(), R, F, DT[dt], st.cuda_stream)}
            for k, fn in calls.items():
                res = []
                for it in range(8):
                    sink.copy_(flush.sum())
                    torch.cuda.synchronize()
                    L.lmbp_trace_act(ctypes.addressof(buf), 0, 1)      # reset
                    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                    e0.record(st)
                    assert fn() == 0
                    e1.record(st)
                    torch.cuda.synchronize()
                    ub = (ctypes.c_ulonglong * (65536 * 2))()
                    nu = L.lmbp_trace_units_act(ctypes.addressof(ub), 65536)
                    n = L.lmbp_trace_act(ctypes.addressof(buf), 8192, 1)
                    r = np.array(buf[:5 * n], dtype=np.float64).reshape(n, 5)
                    t0 = r[:, 1].min()
                    ent, first, ext, tiles = r[:, 1] - t0, r[:, 2] - t0, r[:, 3] - t0, r[:, 4]
                    res.append({"event_us": e0.elapsed_time(e1) * 1e3, "ctas": n, "sms": int(len(set(r[:, 0]))),
                                "span_us": float(ext.max()) / 1e3,
                                "entry_p50_us": float(np.median(ent)) / 1e3, "entry_max_us": float(ent.max()) / 1e3,
                                "first_data_p50_us": float(np.median(first)) / 1e3,
                                "first_data_max_us": float(first.max()) / 1e3,
                                "exit_min_us": float(ext.min()) / 1e3, "exit_p10_us": float(np.percentile(ext, 10)) / 1e3,
                                "exit_p50_us": float(np.median(ext)) / 1e3,
                                "tiles_min": int(tiles.min()), "tiles_max": int(tiles.max()),
                                "tiles_total": int(tiles.sum())})
                    if nu > 0:
                        u = np.array(ub[:2 * nu], dtype=np.float64).reshape(nu, 2)
                        u = u[np.argsort(u[:, 1])]
                        # claim order vs unit index: rank correlation and the index range of the last 5 %
                        order = np.argsort(np.argsort(u[:, 0]))
                        rc = float(np.corrcoef(order, np.arange(nu))[0, 1])
                        tail = u[int(0.95 * nu):, 0]
                        res[-1].update({"claims": int(nu), "claim_order_corr": round(rc, 4),
                                        "last5pct_unit_min": int(tail.min()), "last5pct_unit_max": int(tail.max()),
                                        "units_total": int(u[:, 0].max())})
                med = {kk: round(float(np.median([q[kk] for q in res[2:] if kk in q])), 3) for kk in res[-1]}
                print(json.dumps({"variant": name, "config": cname, "kernel": k, **med}), flush=True)


if __name__ == "__main__":
    main()
