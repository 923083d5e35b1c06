"""Host-side block logic (no GPU): the fine-tuning regimes, Prop. 5.1
condition 3 per regime, the decoded Fig. 5/6 unit model, and
the exact reference blocks' saved bytes on CPU (which linears keep inputs)."""
import pytest
import torch

from paper_2406_16282_b200.blocks import TUNINGS, Block, activation_bytes, linear_modes, saves_input, unit_model


def test_unit_model_reproduces_the_papers_ratios():
    v = unit_model("vit", 4.0)
    assert v["exact_units"] == 19 and v["ours_units"] == 11.5
    assert abs(4 / v["exact_units"] - 0.2105) < 1e-4              # GELU and LN: 21.05 % each
    ll = unit_model("llama", 13824 / 5120)
    assert abs(ll["exact_units"] - 21.8) < 1e-9
    assert abs(2.7 / ll["exact_units"] - 0.1239) < 1e-4 and abs(4 / ll["exact_units"] - 0.1835) < 1e-4
    assert abs(ll["ours_units"] - 15.4375) < 1e-9


def test_condition_3_per_regime():
    want = {"full": (True, True), "lora_qv": (True, False), "lora_all": (True, True),
            "lora_fa_qv": (False, False), "lora_fa_all": (False, False), "frozen_ffn": (True, False)}
    for arch in ("vit", "llama"):
        for t in TUNINGS:
            m = linear_modes(arch, t)
            cons1 = any(saves_input(m[k]) for k in ("q", "k", "v"))
            cons2 = any(saves_input(m[k]) for k in (("fc1",) if arch == "vit" else ("gate", "up")))
            assert (cons1, cons2) == want[t], (arch, t)
    with pytest.raises(ValueError):
        linear_modes("vit", "qlora")


@pytest.mark.parametrize("tuning", TUNINGS)
def test_exact_block_cpu_saved_inputs(tuning):
    b, n, c, h = 2, 8, 32, 128
    blk = Block("vit", c, h, 4, tuning=tuning, device="cpu", norm_fp32=False)
    x = torch.randn(b, n, c, dtype=torch.bfloat16, requires_grad=True)
    _, per = activation_bytes(blk, x, by_module=True)
    R = b * n
    for name, mode in blk.modes.items():
        got = per.get(name, 0)
        r = 2 * R * blk.get_submodule(name).rank if mode in ("lora", "lora_fa") else 0
        if name in ("k", "v") and saves_input(mode) and saves_input(blk.modes["q"]):
            continue                                          # same input as q: counted once, under q
        if name == "proj":
            full_in = 0                                       # its input is SDPA's saved output ([b, n, h, d] layout)
        elif name == "fc2":
            full_in = 2 * R * h
        else:
            full_in = 2 * R * c
        assert got == (full_in if saves_input(mode) else 0) + r, (name, mode, got)
    out = blk(x)
    out.float().sum().backward()
    assert x.grad is not None and torch.isfinite(x.grad.float()).all()
