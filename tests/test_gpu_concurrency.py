"""Reentrancy ("no global mutable state ... reentrant across host
threads, streams and devices"): several host threads drive every kernel
family through the C ABI at once, each on its own stream with its own
buffers and its own shapes (so the per-kernel first-launch work -- shared-
memory attributes, occupancy caches -- races too), repeatedly; every result
must be bitwise identical to the same call run alone and in order."""
import threading

import numpy as np
import pytest
import torch

import synth
import paper_2406_16282_b200 as P
from paper_2406_16282_b200 import tables
from test_gpu_parity import DEV, st

pytestmark = pytest.mark.gpu


def _jobs():
    """(name, fn(stream) -> tuple of output tensors); inputs built once."""
    jobs = []
    for i, (dt, R, F, H) in enumerate([("bf16", 96, 11008, 4096), ("f16", 33, 3072, 768), ("f32", 17, 4099, 5120),
                                       ("bf16", 5, 40000, 40000)]):
        x = synth.act_input(R, F, dt, mode="coverage").to(DEV)
        dy = synth.grad_input(R, F, dt).to(DEV)
        xn = synth.norm_input(R, H, dt).to(DEV)
        gn = synth.grad_input(R, H, dt, stream=synth.S_NORM_DY).to(DEV)

        def act(s, x=x, dy=dy):
            y, c = P.resilu2_fwd(x, stream=s)
            y2, c2 = P.regelu2_fwd(x, stream=s)
            return y, c, P.resilu2_bwd(dy, c, stream=s), y2, c2, P.regelu2_bwd(dy, c2, stream=s)

        def norm(s, xn=xn, gn=gn):
            yl, rl = P.msln_fwd(xn, 1e-6, stream=s)
            yr, rr = P.msrms_fwd(xn, 1e-6, stream=s)
            return yl, rl, P.msln_bwd(gn, yl, rl, stream=s), yr, rr, P.msrms_bwd(gn, yr, rr, stream=s)

        def kbit(s, x=x, dy=dy):
            out = []
            for k, thr, lv in ((2, tables.REGELU2["c"], tables.levels(tables.REGELU2)),
                               (3, [-3.0 + i for i in range(7)], [j / 7 for j in range(8)]),
                               (4, [-3.0 + 0.4 * i for i in range(15)], [j / 15 for j in range(16)])):
                for act in ("gelu", "silu"):
                    y, c = P.stepact_fwd(x, act, k, thr, stream=s)
                    out += [y, c, P.stepact_bwd(dy, c, k, lv, stream=s)]
            return tuple(out)

        def swiglu(s, x=x, dy=dy):
            h, a, c = P.reswiglu2_fwd(x, dy, stream=s)
            dg, du = P.reswiglu2_bwd(dy, dy, a, c, stream=s)
            return h, a, c, dg, du

        jobs += [(f"act{i}", act), (f"norm{i}", norm), (f"kbit{i}", kbit), (f"swiglu{i}", swiglu)]
        if dt != "f32":
            def mixed(s, xn=xn, gn=gn, t=xn.dtype):
                ym, rm = P.msrms_fwd_mixed(xn.float(), 1e-6, t, stream=s)
                return ym, rm, P.msrms_bwd_mixed(gn, ym, rm, stream=s)
            jobs.append((f"mixed{i}", mixed))
    return jobs


def _bytes(outs):
    return [np.ascontiguousarray(st(o)).tobytes() for o in outs]


def run(concurrent_first: bool) -> None:
    jobs = _jobs()
    got, errors = {}, []

    def worker(tid):
        try:
            s = torch.cuda.Stream()
            for rep in range(3):
                for name, fn in jobs[tid::4]:
                    with torch.cuda.stream(s):
                        outs = fn(s.cuda_stream)
                    s.synchronize()
                    got[(name, rep)] = _bytes(outs)
        except Exception as e:  # surfaced in the main thread
            errors.append(repr(e))

    def concurrent():
        threads = [threading.Thread(target=worker, args=(t,)) for t in range(4)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()

    if concurrent_first:          # the threads also race on every kernel's first launch
        concurrent()
    ref = {}                      # one after another on the current stream
    for name, fn in jobs:
        outs = fn(torch.cuda.current_stream().cuda_stream)
        torch.cuda.synchronize()
        ref[name] = _bytes(outs)
    if not concurrent_first:
        concurrent()
    assert not errors, errors
    for (name, rep), b in got.items():
        assert b == ref[name], f"{name} (repeat {rep}) differs under concurrency"
    assert len(got) == 3 * len(jobs)


def test_threads_and_streams_bitwise():
    run(concurrent_first=False)


def test_threads_race_on_first_launch():
    """In a fresh process: the four threads launch every kernel for the first
    time concurrently (per-kernel attribute and occupancy setup included)."""
    import os
    import subprocess
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    r = subprocess.run([sys.executable, os.path.abspath(__file__)], cwd=os.path.dirname(here),
                       capture_output=True, text=True, timeout=600,
                       env=dict(os.environ, PYTHONPATH=os.pathsep.join([os.path.dirname(here), here])))
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]


if __name__ == "__main__":
    run(concurrent_first=True)
    print("concurrent-first ok")
