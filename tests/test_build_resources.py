"""Guards on the compiled kernels' resources (ptxas -v logs written by the
build): the pipelined kernels' register counts decide how many CTAs fit per
SM, and a silent jump (e.g. a changed __launch_bounds__) cost 9 % before.
Skipped when the build logs are absent."""
import os
import re
import subprocess

import pytest

OBJ = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2406_16282_b200", "_obj")


def regs(log):
    out = {}
    text = open(os.path.join(OBJ, log)).read()
    for m in re.finditer(r"Compiling entry function '([^']+)'.*?Used (\d+) registers", text, re.S):
        out[m.group(1)] = int(m.group(2))
    return out


def demangle(names):
    r = subprocess.run(["c++filt"], input="\n".join(names), capture_output=True, text=True)
    return dict(zip(names, r.stdout.splitlines()))


@pytest.mark.skipif(not os.path.exists(os.path.join(OBJ, "act.ptxas.log")), reason="no build logs")
def test_pipeline_register_budgets():
    r = regs("act.ptxas.log")
    d = demangle(list(r))
    by = {d[k]: v for k, v in r.items()}
    fwd = [v for k, v in by.items() if "ActFwdOp<__nv_bfloat16, 1" in k]
    bwd = [v for k, v in by.items() if "ActBwdOp<__nv_bfloat16" in k]
    assert fwd and bwd
    # SiLU 16-bit forward CTA = 17 warps (544 threads): 2 CTAs / SM need <= 60 registers
    assert max(fwd) <= 60, by
    # backward CTA = 13 warps (416 threads): 2 CTAs / SM need <= 78 registers
    assert max(bwd) <= 78, by


@pytest.mark.skipif(not os.path.exists(os.path.join(OBJ, "norm.ptxas.log")), reason="no build logs")
def test_no_spills_in_hot_kernels():
    for log in ("act.ptxas.log", "swiglu.ptxas.log"):
        text = open(os.path.join(OBJ, log)).read()
        spills = [int(x) for x in re.findall(r"(\d+) bytes spill stores", text)]
        assert max(spills) == 0, log


@pytest.mark.skipif(not os.path.exists(os.path.join(OBJ, "stepact.ptxas.log")), reason="no build logs")
def test_kbit_forward_register_budget():
    """16-bit step forwards read y from the 128 KB table (one CTA of 17 warps
    per SM: <= 120 registers); fp32 k = 4 keeps 2 CTAs / SM (<= 60); no step
    forward spills."""
    r = regs("stepact.ptxas.log")
    d = demangle(list(r))
    by = {d[k]: v for k, v in r.items()}
    k16 = [v for k, v in by.items() if re.search(r"StepFwdOp<(__nv_bfloat16|__half), 0, false, [1234]>", k)]
    silu4 = [v for k, v in by.items() if re.search(r"StepFwdOp<(__nv_bfloat16|__half), 1, false, 4>", k)]
    k32 = [v for k, v in by.items() if re.search(r"StepFwdOp<float, [01], true, 4>", k)]
    assert len(k16) == 8 and len(silu4) == 2 and len(k32) == 2, by
    # GELU 16-bit reads the table (1 CTA / SM: <= 120); SiLU k = 4 keeps 3 x 416-thread CTAs (<= 52)
    assert max(k16) <= 120 and max(silu4) <= 52 and max(k32) <= 60, by
    text = open(os.path.join(OBJ, "stepact.ptxas.log")).read()
    for m in re.finditer(r"Function properties for (\S+)\n.*?(\d+) bytes spill stores", text):
        if "StepFwdOp" in demangle([m.group(1)])[m.group(1)]:
            assert int(m.group(2)) == 0, m.group(1)


@pytest.mark.skipif(not os.path.exists(os.path.join(OBJ, "act.ptxas.log")), reason="no build logs")
def test_lut_forward_fits_one_cta_per_sm():
    """The 16-bit forward (ActFwdLutOp): 544-thread CTAs, one per SM next to
    its 128 KB table, so <= 120 registers."""
    r = regs("act.ptxas.log")
    d = demangle(list(r))
    lut = [v for k, v in d.items() if "ActFwdLutOp" in v]
    assert len(lut) == 2                          # GELU bf16 / fp16 (kUseLut)
    assert max(r[k] for k, v in d.items() if "ActFwdLutOp" in v) <= 120


@pytest.mark.skipif(not os.path.exists(os.path.join(OBJ, "norm.ptxas.log")), reason="no build logs")
def test_norm_row_pipeline_does_not_spill():
    """norm_row_tma runs 544-thread CTAs (~120 registers per thread): only
    V <= 4 instantiations exist and none spills."""
    text = open(os.path.join(OBJ, "norm.ptxas.log")).read()
    seen = 0
    for m in re.finditer(r"Function properties for (\S+)\n.*?(\d+) bytes spill stores", text):
        name = demangle([m.group(1)])[m.group(1)]
        if "norm_row_tma" in name:
            seen += 1
            assert int(m.group(2)) == 0, name
    assert seen > 0
