#!/bin/bash
# 16-bit forward: correctly rounded shared-memory table (ActFwdLutOp) vs the polynomial/MUFU math (LMBP_NO_LUT)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_*.so; do n=$(basename $f .so); n=${n#liblmbp_}; V="$V ${n%%-*}:@$f"; done
for c in c2 c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,step2_fwd,step4_fwd,copy --variants $V --iters 30; done > gpurun_out/sweep37.jsonl 2> gpurun_out/sweep37.err
cat gpurun_out/sweep37.jsonl
