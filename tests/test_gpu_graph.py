"""CUDA-graph capture of the C-ABI launches (DESIGN 5.10: the launches carry
the programmatic-stream-serialization attribute, which capture turns into
programmatic graph edges).  A graph of a whole step -- every kernel family,
each consuming the previous one's output -- recorded once and replayed on new
input contents must give the same bytes as the eager calls."""
import pytest
import torch

import synth
import paper_2406_16282_b200 as P
from test_gpu_parity import DEV

pytestmark = pytest.mark.gpu


def _buffers(R, F, H, dt):
    x = torch.empty(R, F, dtype=synth.TORCH_DTYPES[dt], device=DEV)
    d = {"x": x, "dy": torch.empty_like(x), "xn": torch.empty(R, H, dtype=x.dtype, device=DEV)}
    d["gn"] = torch.empty_like(d["xn"])
    d["y"], d["dx"], d["h"], d["a"], d["dg"], d["du"], d["y4"], d["dx4"] = (torch.empty_like(x) for _ in range(8))
    d["codes"] = torch.empty(P.codes_bytes(R * F), dtype=torch.uint8, device=DEV)
    d["cs"] = torch.empty_like(d["codes"])
    d["c4"] = torch.empty(P.codes_bytes_k(R * F, 4), dtype=torch.uint8, device=DEV)
    d["yn"], d["dxn"] = torch.empty_like(d["xn"]), torch.empty_like(d["xn"])
    d["rstd"] = torch.empty(R, dtype=torch.float32, device=DEV)
    return d


THR4 = [-3.0 + 0.4 * i for i in range(15)]
LV4 = [i / 15 for i in range(16)]


def _step(b, act, norm):
    fwd, bwd = (P.regelu2_fwd, P.regelu2_bwd) if act == "gelu" else (P.resilu2_fwd, P.resilu2_bwd)
    nf, nb = (P.msln_fwd, P.msln_bwd) if norm == "ln" else (P.msrms_fwd, P.msrms_bwd)
    nf(b["xn"], 1e-6, y=b["yn"], rstd=b["rstd"])
    fwd(b["x"], y=b["y"], codes=b["codes"])
    bwd(b["dy"], b["codes"], dx=b["dx"])
    nb(b["gn"], b["yn"], b["rstd"], dx=b["dxn"])
    P.reswiglu2_fwd(b["x"], b["dy"], h=b["h"], a=b["a"], codes=b["cs"])
    P.reswiglu2_bwd(b["dx"], b["dy"], b["a"], b["cs"], dgate=b["dg"], dup=b["du"])
    P.stepact_fwd(b["h"], act, 4, THR4, y=b["y4"], codes=b["c4"])
    P.stepact_bwd(b["du"], b["c4"], 4, LV4, dx=b["dx4"])


def _fill(b, R, F, H, dt, row0):
    b["x"].copy_(synth.act_input(R, F, dt, mode="coverage", row_start=row0))
    b["dy"].copy_(synth.grad_input(R, F, dt, row_start=row0))
    b["xn"].copy_(synth.norm_input(R, H, dt, row_start=row0))
    b["gn"].copy_(synth.grad_input(R, H, dt, row_start=row0, stream=synth.S_NORM_DY))


OUT = ("y", "codes", "dx", "yn", "rstd", "dxn", "h", "a", "cs", "dg", "du", "y4", "c4", "dx4")


@pytest.mark.parametrize("dt,act,norm", [("bf16", "gelu", "ln"), ("bf16", "silu", "rms"), ("f32", "silu", "ln"),
                                         ("f16", "gelu", "rms")])
def test_graph_replay_equals_eager(dt, act, norm):
    R, F, H = 300, 3072, 768
    g_buf, e_buf = _buffers(R, F, H, dt), _buffers(R, F, H, dt)
    _fill(g_buf, R, F, H, dt, 0)
    _step(g_buf, act, norm)                 # first launches (attributes, occupancy caches) outside capture
    torch.cuda.synchronize()
    graph = torch.cuda.CUDAGraph()
    with torch.cuda.graph(graph):
        _step(g_buf, act, norm)
    for row0 in (0, 4096, 70000):           # new contents in the captured buffers, then replay
        _fill(g_buf, R, F, H, dt, row0)
        graph.replay()
        _fill(e_buf, R, F, H, dt, row0)
        _step(e_buf, act, norm)
        torch.cuda.synchronize()
        for k in OUT:
            u = g_buf[k].reshape(-1).view(torch.uint8)
            v = e_buf[k].reshape(-1).view(torch.uint8)
            assert torch.equal(u, v), (k, row0)
