#!/bin/bash
# row-pipeline work unit (rows per CLC request) for the norm backward at C4 / C5 / C3-bf16-free configs
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels norm_bwd --iters 30 --variants u1:LMBP_ROW_UNIT=1 u2:LMBP_ROW_UNIT=2 u4:LMBP_ROW_UNIT=4 head:@paper_2406_16282_b200/liblmbp.so; done > gpurun_out/sweep29.jsonl 2> gpurun_out/sweep29.err
cat gpurun_out/sweep29.jsonl; tail -3 gpurun_out/sweep29.err
