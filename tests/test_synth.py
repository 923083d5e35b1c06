"""Seeded generators: slice invariance (any row range reproduces the same rows
of the full tensor -- what row sharding across ranks relies on)."""
import torch

import synth


def test_slice_invariance_cpu():
    full = synth.act_input(700, 33, "bf16", mode="coverage")
    part = synth.act_input(300, 33, "bf16", row_start=250, mode="coverage")
    assert torch.equal(full[250:550].view(torch.int16), part.view(torch.int16))
    nf = synth.norm_input(600, 17, "f32")
    npart = synth.norm_input(100, 17, "f32", row_start=255)
    assert torch.equal(nf[255:355], npart)
    r = synth.rstd_input(600)
    assert torch.equal(r[512:600], synth.rstd_input(88, row_start=512))
    assert float(r.min()) >= 0.5 and float(r.max()) <= 2.0


def test_streams_independent_and_deterministic():
    a = synth.act_input(64, 64, "f32")
    b = synth.grad_input(64, 64, "f32")
    assert not torch.equal(a, b)
    assert torch.equal(a, synth.act_input(64, 64, "f32"))


def test_configs_match_baseline():
    import json, os
    bj = json.load(open(os.path.join(os.path.dirname(__file__), "..", "BASELINE.json")))
    assert len(bj["configs"]) == 5
    c = synth.CONFIGS
    assert (c["c1"]["R"], c["c1"]["F"], c["c1"]["H"]) == (394, 3072, 768)
    assert (c["c4"]["R"], c["c4"]["F"], c["c4"]["H"]) == (8192, 11008, 4096)
    assert (c["c5"]["R"], c["c5"]["F"], c["c5"]["H"]) == (32768, 13824, 5120)
