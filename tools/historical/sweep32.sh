#!/bin/bash
# k-bit step forward pipeline shape (LMBP_STEP_W/U/S, LMBP_STEP_MINB4) at C4 / C5
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V="head:@paper_2406_16282_b200/liblmbp.so sa:LMBP_STEP_W=8,LMBP_STEP_U=4,LMBP_STEP_S=4 sc:LMBP_STEP_W=16,LMBP_STEP_U=1,LMBP_STEP_S=4 sd:LMBP_STEP_W=16,LMBP_STEP_U=2,LMBP_STEP_S=3 se:LMBP_STEP_W=12,LMBP_STEP_U=2,LMBP_STEP_S=4,LMBP_STEP_MINB4=3 sf:LMBP_STEP_W=16,LMBP_STEP_U=2,LMBP_STEP_S=4,LMBP_STEP_MINB4=1 sg:LMBP_STEP_W=8,LMBP_STEP_U=2,LMBP_STEP_S=4,LMBP_STEP_MINB4=4"
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels step4_fwd,step2_fwd --iters 30 --variants $V; done > gpurun_out/sweep32.jsonl 2> gpurun_out/sweep32.err
cat gpurun_out/sweep32.jsonl; tail -3 gpurun_out/sweep32.err
