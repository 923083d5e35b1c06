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
    fwd = [v for k, v in by.items() if "ActFwdOp<__nv_bfloat16" in k]
    bwd = [v for k, v in by.items() if "ActBwdOp<__nv_bfloat16" in k]
    assert fwd and bwd
    # forward CTA = 17 warps (544 threads): 2 CTAs / SM need <= 60 registers
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
    """k = 4 SiLU forward, 16-bit types: 13-warp CTAs (416 threads), 3 per SM
    need <= 52 registers (ptxas targets 48); no step forward spills (sweep33)."""
    r = regs("stepact.ptxas.log")
    d = demangle(list(r))
    by = {d[k]: v for k, v in r.items()}
    k4 = [v for k, v in by.items() if re.search(r"StepFwdOp<(__nv_bfloat16|__half), 1, false, 4>", k)]
    assert len(k4) == 2, by
    assert max(k4) <= 52, by
    text = open(os.path.join(OBJ, "stepact.ptxas.log")).read()
    for m in re.finditer(r"Function properties for (\S+)\n.*?(\d+) bytes spill stores", text):
        if "StepFwdOp" in demangle([m.group(1)])[m.group(1)]:
            assert int(m.group(2)) == 0, m.group(1)


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
