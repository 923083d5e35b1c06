"""PCIe ceiling for bench's e2e: pinned H2D alone, D2H alone, and both at
once on two streams (256 MB buffers, CUDA events, best of 5)."""
import json
import torch

N = 256 << 20
h_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def best(fn, nbytes):
    out = []
    for _ in range(6):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        out.append(nbytes / (e0.elapsed_time(e1) / 1e3) / 1e9)
    return round(max(out[1:]), 1)


def both():
    cur = torch.cuda.current_stream()
    ev = torch.cuda.Event()
    ev.record(cur)
    s1.wait_event(ev)
    s2.wait_event(ev)
    with torch.cuda.stream(s1):
        d_in.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_out, non_blocking=True)
    for s in (s1, s2):
        e = torch.cuda.Event()
        e.record(s)
        cur.wait_event(e)


print(json.dumps({"h2d_GBs": best(lambda: d_in.copy_(h_in, non_blocking=True), N),
                  "d2h_GBs": best(lambda: h_out.copy_(d_out, non_blocking=True), N),
                  "bidirectional_GBs": best(both, 2 * N)}))
