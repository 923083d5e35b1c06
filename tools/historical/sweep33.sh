#!/bin/bash
# k = 4 step forward: consumer warps x CTAs per SM (register cap) around sweep32's best
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V="head:@paper_2406_16282_b200/liblmbp.so t12m3:LMBP_STEP4_W=12,LMBP_STEP_MINB4=3 t10m4:LMBP_STEP4_W=10,LMBP_STEP_MINB4=4 t12m3s3:LMBP_STEP4_W=12,LMBP_STEP4_S=3,LMBP_STEP_MINB4=3 t8m5:LMBP_STEP4_W=8,LMBP_STEP_MINB4=5 t14m3:LMBP_STEP4_W=14,LMBP_STEP_MINB4=3 t16m2:LMBP_STEP4_W=16,LMBP_STEP_MINB4=2"
for c in c4 c5 c3; do timeout 600 python tools/sweep.py --config $c --kernels step4_fwd --iters 30 --variants $V; done > gpurun_out/sweep33.jsonl 2> gpurun_out/sweep33.err
cat gpurun_out/sweep33.jsonl; tail -3 gpurun_out/sweep33.err
