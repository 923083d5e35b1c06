"""Where the in-stream step loses time between kernels (DESIGN 5.10): for one
config, time from CUDA graphs (a) each step kernel alone, back to back with
itself, and (b) each consecutive pair of the step (A then B, repeated),
rotating over bench.py's stream-protocol buffer sets.  The
transition cost of A -> B is t(AB) - t(A) - t(B) per pair.

    python tools/stream_pairs.py --config c2
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import bench  # noqa: E402
import synth  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c2")
    ap.add_argument("--reps", type=int, default=40)
    a = ap.parse_args()
    import paper_2406_16282_b200 as P
    dev = torch.device("cuda", 0)
    torch.cuda.set_device(dev)
    cfg = synth.CONFIGS[a.config]
    stream = torch.cuda.current_stream(dev)
    w = bench.Workload(P, cfg, 0, cfg["R"], dev, stream, 1e-6)
    n = bench.stream_sets(w.nbytes, torch.cuda.get_device_properties(dev).L2_cache_size)
    sw = bench.StreamWorkload(w, n)
    K = bench.KERNELS
    single = {k: sw.timed_graph(lambda i, k=k: sw.launch[k](i % n), sw.per_graph(8), a.reps * 8, 16, 1) * 1e3
              for k in K}
    pairs = {}
    for i in range(len(K)):
        A, B = K[i], K[(i + 1) % len(K)]

        def body(j, A=A, B=B):
            s = j // 2       # B on the next set: it never reads what A just wrote
            sw.launch[A](s % n) if j % 2 == 0 else sw.launch[B]((s + 1) % n)
        t = 2 * sw.timed_graph(body, 2 * sw.per_graph(4), a.reps * 8, 16, 1) * 1e3   # us per (A, B) pair
        pairs[f"{A}->{B}"] = {"pair_us": round(t, 2), "transition_us": round(t - single[A] - single[B], 2)}
    step = sw.timed_graph(sw.step, sw.per_graph(2), a.reps * 2, 4, 1) * 1e3
    print(json.dumps({"config": a.config, "buffer_sets": n, "single_us": {k: round(v, 2) for k, v in single.items()},
                      "pairs": pairs, "step_us": round(step, 2),
                      "step_minus_singles_us": round(step - sum(single.values()), 2)}))


if __name__ == "__main__":
    main()
