#!/bin/bash
# k = 4 SiLU forward: first level-0 mux stage on the FMA pipe (bf16x2 m a + (1 - m) b) vs all-LOP3
# (historical: the LMBP_STEP_FMA_MUX knob was removed after this sweep; see profiles/README.md)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels step4_fwd --iters 30 --variants head:@paper_2406_16282_b200/liblmbp.so fmux:LMBP_STEP_FMA_MUX head2:@paper_2406_16282_b200/liblmbp.so; done > gpurun_out/sweep35.jsonl 2> gpurun_out/sweep35.err
cat gpurun_out/sweep35.jsonl; tail -3 gpurun_out/sweep35.err
