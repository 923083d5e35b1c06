#!/bin/bash
# k-bit step forward: final shape (new) vs the previous library (old) at C2-C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c5 c3 c2; do timeout 600 python tools/sweep.py --config $c --kernels step4_fwd,step4_bwd,step2_fwd --iters 30 --variants old:@paper_2406_16282_b200/_variants/old_lmbp.so new:@paper_2406_16282_b200/liblmbp.so; done > gpurun_out/sweep34.jsonl 2> gpurun_out/sweep34.err
cat gpurun_out/sweep34.jsonl; tail -3 gpurun_out/sweep34.err
