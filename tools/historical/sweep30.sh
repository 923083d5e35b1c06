#!/bin/bash
# row pipeline shape for the norm backward: vectors per thread (VAIM) x ring budget (STAGE_KB)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels norm_bwd --iters 30 --variants v4s96:LMBP_ROW_VAIM=4,LMBP_ROW_STAGE_KB=96 v2s96:LMBP_ROW_VAIM=2,LMBP_ROW_STAGE_KB=96 v8s96:LMBP_ROW_VAIM=8,LMBP_ROW_STAGE_KB=96 v4s48:LMBP_ROW_VAIM=4,LMBP_ROW_STAGE_KB=48 v2s48:LMBP_ROW_VAIM=2,LMBP_ROW_STAGE_KB=48 v4s64:LMBP_ROW_VAIM=4,LMBP_ROW_STAGE_KB=64 v4s96b:LMBP_ROW_VAIM=4,LMBP_ROW_STAGE_KB=96; done > gpurun_out/sweep30.jsonl 2> gpurun_out/sweep30.err
cat gpurun_out/sweep30.jsonl; tail -3 gpurun_out/sweep30.err
