"""Programmatic dependent launch (csrc/common.cuh): every hot-path kernel may
be scheduled before its predecessor on the stream has finished and waits
(griddepcontrol.wait) before its first global access.  These chains make each
launch depend on the one before it in both directions -- it reads what the
previous kernel wrote (RAW) and overwrites what the previous kernel read
(WAR) -- and run them back to back, and again with a device synchronisation
after every launch (no predecessor in flight, so nothing can overlap); the
results must be bitwise identical.  A torch kernel writing a buffer right
before a launch that reads it is covered too (a predecessor that never
triggers early), and a subprocess with LMBP_PDL=0 (plain stream order) must
give the same bytes."""
import os
import subprocess
import sys

import numpy as np
import pytest
import torch

import synth
import paper_2406_16282_b200 as P
from test_gpu_parity import DEV

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _chain(dt, R, F, H, iters, sync, seed_rows=0):
    """Act and norm chains in which every launch consumes the previous one's
    output and overwrites the previous one's input.  Returns numpy bytes."""
    a = synth.act_input(R, F, dt, mode="coverage", row_start=seed_rows).to(DEV)
    b = torch.empty_like(a)
    codes = torch.empty(P.codes_bytes(R * F), dtype=torch.uint8, device=DEV)
    p = synth.norm_input(R, H, dt, row_start=seed_rows).to(DEV)
    q, r = torch.empty_like(p), torch.empty_like(p)
    rstd = torch.empty(R, dtype=torch.float32, device=DEV)
    s = torch.cuda.current_stream(DEV)
    fences = []
    for i in range(iters):
        fwd, bwd = (P.regelu2_fwd, P.regelu2_bwd) if i % 2 == 0 else (P.resilu2_fwd, P.resilu2_bwd)
        nf, nb = (P.msln_fwd, P.msln_bwd) if i % 2 == 0 else (P.msrms_fwd, P.msrms_bwd)
        steps = [
            lambda: fwd(a, y=b, codes=codes, stream=s),             # reads a, writes b, codes
            lambda: bwd(b, codes, dx=a, stream=s),                  # reads b, codes (RAW); writes a (WAR)
            lambda: nf(p, 1e-6, y=q, rstd=rstd, stream=s),          # reads p, writes q, rstd
            lambda: nb(q, q, rstd, dx=r, stream=s),                 # reads q, rstd (RAW); writes r
            lambda: nf(r, 1e-6, y=p, rstd=rstd, stream=s),          # reads r (RAW); writes p, rstd (WAR)
        ]
        for st in steps:
            st()
            if sync:
                torch.cuda.synchronize()
        fences.append(a.view(torch.uint8).sum(dtype=torch.int64))  # a torch reader between our launches
    torch.cuda.synchronize()
    return [t.cpu().view(torch.uint8).numpy().copy() for t in (a, b, codes, p, q, r, rstd)], \
        [int(f) for f in fences]


@pytest.mark.parametrize("dt,R,F,H", [("bf16", 512, 3072, 768), ("f32", 37, 11008, 4096),
                                      ("f16", 1, 40000, 40000)])
def test_pdl_chain_equals_serialised(dt, R, F, H):
    back, fb = _chain(dt, R, F, H, iters=12, sync=False)
    ser, fs = _chain(dt, R, F, H, iters=12, sync=True)
    for i, (u, v) in enumerate(zip(back, ser)):
        assert np.array_equal(u, v), f"output {i} differs between back-to-back and serialised launches"
    assert fb == fs


def _chain_other(iters, sync):
    """The other kernel families (k-bit step activations, fused ReSwiGLU2,
    mixed-precision MS norms) in one dependent chain."""
    from paper_2406_16282_b200 import tables
    R, F, H = 129, 11008, 4096
    x = synth.act_input(R, F, "bf16", mode="coverage").to(DEV)
    u = synth.grad_input(R, F, "bf16").to(DEV)
    y = torch.empty_like(x)
    k3 = P.codes_bytes_k(R * F, 3)
    c3 = torch.empty(k3, dtype=torch.uint8, device=DEV)
    h, act = torch.empty_like(x), torch.empty_like(x)
    cs = torch.empty(P.codes_bytes(R * F), dtype=torch.uint8, device=DEV)
    dg, du = torch.empty_like(x), torch.empty_like(x)
    r32 = synth.norm_input(R, H, "f32").to(DEV)
    yb = torch.empty(R, H, dtype=torch.bfloat16, device=DEV)
    rstd = torch.empty(R, dtype=torch.float32, device=DEV)
    thr, lv = [-3.0 + i for i in range(7)], [j / 7 for j in range(8)]
    s = torch.cuda.current_stream(DEV)
    steps = [
        lambda: P.stepact_fwd(x, "silu", 3, thr, y=y, codes=c3, stream=s),      # x -> y, c3
        lambda: P.stepact_bwd(y, c3, 3, lv, dx=x, stream=s),                     # y, c3 -> x (WAR on x)
        lambda: P.reswiglu2_fwd(x, u, h=h, a=act, codes=cs, stream=s),          # x, u -> h, a, codes
        lambda: P.reswiglu2_bwd(h, u, act, cs, dgate=dg, dup=x, stream=s),      # h, a, codes -> dg, x (WAR)
        lambda: P.msrms_fwd_mixed(r32, 1e-6, torch.bfloat16, y=yb, rstd=rstd, stream=s),
        lambda: P.msrms_bwd_mixed(yb, yb, rstd, dx=r32, stream=s),              # yb, rstd -> r32 (WAR)
    ]
    for _ in range(iters):
        for st in steps:
            st()
            if sync:
                torch.cuda.synchronize()
    torch.cuda.synchronize()
    return [t.cpu().view(torch.uint8).numpy().copy() for t in (x, y, c3, h, act, cs, dg, r32, yb, rstd)]


def test_pdl_chain_other_families():
    for i, (u, v) in enumerate(zip(_chain_other(4, False), _chain_other(4, True))):
        assert np.array_equal(u, v), f"output {i} differs between back-to-back and serialised launches"


def test_pdl_after_torch_writer():
    """A torch kernel fills the input right before each launch; the launch
    must see the new contents (griddepcontrol.wait before the first load)."""
    R, F = 256, 3072
    src = [synth.act_input(R, F, "bf16", mode="coverage", row_start=r).to(DEV) for r in (0, R, 2 * R)]
    x = torch.empty_like(src[0])
    outs = []
    for i in range(9):
        x.copy_(src[i % 3])
        y, c = P.regelu2_fwd(x)
        outs.append((y.clone(), c.clone()))
    torch.cuda.synchronize()
    for i, (y, c) in enumerate(outs):
        y_ref, c_ref = P.regelu2_fwd(src[i % 3])
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int16), y_ref.view(torch.int16)) and torch.equal(c, c_ref), i


_SUB = r"""
import sys, numpy as np
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
from test_gpu_pdl import _chain
outs, fences = _chain("bf16", 300, 3072, 768, iters=6, sync=False)
np.savez({path!r}, *outs, fences=np.array(fences))
"""


def test_pdl_off_gives_same_bytes(tmp_path):
    outs = []
    for pdl in ("0", "1"):
        path = str(tmp_path / f"pdl{pdl}.npz")
        env = dict(os.environ, LMBP_PDL=pdl)
        code = _SUB.format(root=ROOT, tests=os.path.join(ROOT, "tests"), path=path)
        r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
        assert r.returncode == 0, r.stderr[-2000:]
        outs.append(np.load(path))
    for k in outs[0].files:
        assert np.array_equal(outs[0][k], outs[1][k]), k


def test_pdl_honours_cross_stream_event():
    """Stream A: our kernel, then a wait on an event of stream B, then our
    kernel reading what B wrote.  The second launch follows a kernel on A, but
    the event is a dependency too: it must see B's bytes, however long B
    takes (B is made slow: many large copies before the write that matters)."""
    R, F = 64, 3072
    a, b = torch.cuda.Stream(DEV), torch.cuda.Stream(DEV)
    x1 = synth.act_input(R, F, "bf16", mode="coverage").to(DEV)
    new = synth.act_input(R, F, "bf16", mode="coverage", row_start=R).to(DEV)
    big_src = torch.ones(64 << 20, dtype=torch.float32, device=DEV)
    big_dst = torch.empty_like(big_src)
    y_ref, c_ref = P.regelu2_fwd(new)
    torch.cuda.synchronize()
    for trial in range(5):
        x2 = torch.zeros_like(new)
        torch.cuda.synchronize()
        with torch.cuda.stream(b):
            for _ in range(8):                    # ~2 GB of copies: B finishes long after A's first kernel
                big_dst.copy_(big_src)
            x2.copy_(new)
            ev = torch.cuda.Event()
            ev.record(b)
        with torch.cuda.stream(a):
            P.regelu2_fwd(x1)
            a.wait_event(ev)
            y2, c2 = P.regelu2_fwd(x2)
        torch.cuda.synchronize()
        assert torch.equal(y2.view(torch.int16), y_ref.view(torch.int16)) and torch.equal(c2, c_ref), trial
