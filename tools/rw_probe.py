"""HBM read / write asymmetry probe (B200): times pure-read (sum), pure-write
(fill), copy (1:1) and the two mixes of the activation kernels with torch
kernels, L2 flushed (read of 2 x L2) before every launch, CUDA events on the
launching stream.  Prints one JSON line per probe: bytes read / written, us,
GB/s.  Used to fit a per-direction cost model (DESIGN 5.3).

    python tools/rw_probe.py [--mb 180] [--iters 30]
"""
import argparse
import json

import torch


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mb", type=float, default=180.355072)   # one C4 act tensor (8192 x 11008 bf16)
    ap.add_argument("--iters", type=int, default=30)
    a = ap.parse_args()
    dev = torch.device("cuda")
    n = int(a.mb * 1e6) // 2
    x = torch.randn(n, device=dev).to(torch.bfloat16)
    x2 = torch.randn(n, device=dev).to(torch.bfloat16)
    y = torch.empty_like(x)
    y2 = torch.empty_like(x)
    acc = torch.empty((), dtype=torch.float32, device=dev)
    flush = torch.ones((2 * torch.cuda.get_device_properties(dev).L2_cache_size) // 4, device=dev)
    sink = torch.zeros((), device=dev)
    st = torch.cuda.current_stream()
    B = 2 * n
    probes = {
        "read (sum)": (lambda: torch.sum(x, dim=0, dtype=torch.float32, out=acc), B, 0),
        "write (fill)": (lambda: y.fill_(1.0), 0, B),
        "copy 1:1": (lambda: y.copy_(x), B, B),
        "add 2:1": (lambda: torch.add(x, x2, out=y), 2 * B, B),
        "write 2 (fill x2)": (lambda: (y.fill_(1.0), y2.fill_(1.0)), 0, 2 * B),
    }
    for name, (fn, rd, wr) in probes.items():
        for _ in range(3):
            fn()
        ts = []
        for _ in range(a.iters):
            sink.copy_(flush.sum())
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            fn()
            e1.record(st)
            ts.append((e0, e1))
        torch.cuda.synchronize()
        us = sorted(e0.elapsed_time(e1) * 1e3 for e0, e1 in ts)
        med = us[len(us) // 2]
        print(json.dumps({"probe": name, "read_B": rd, "write_B": wr, "us_med": round(med, 2),
                          "us_min": round(us[0], 2), "GB/s": round((rd + wr) / med / 1e3, 1)}), flush=True)


if __name__ == "__main__":
    main()
