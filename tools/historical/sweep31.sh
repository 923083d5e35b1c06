#!/bin/bash
# SiLU max(x, 0) on the FMA pipe (0.5 x + 0.5 |x|, exact for 16-bit inputs) instead of FMNMX on the ALU pipe
# (historical: the LMBP_SILU_FMA_MAX knob was removed after this sweep; see profiles/README.md)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,step4_fwd,step2_fwd --iters 30 --variants head:@paper_2406_16282_b200/liblmbp.so fmax:LMBP_SILU_FMA_MAX head2:@paper_2406_16282_b200/liblmbp.so; done > gpurun_out/sweep31.jsonl 2> gpurun_out/sweep31.err
cat gpurun_out/sweep31.jsonl; tail -3 gpurun_out/sweep31.err
