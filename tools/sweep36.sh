#!/bin/bash
# static-prefix fraction of the elementwise pipeline (LMBP_EW_STATIC, ew_pipeline.cuh)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_s*.so; do n=$(basename $f .so); n=${n#liblmbp_}; V="$V ${n%%-*}:@$f"; done
for c in c4 c2 c5 c3 c1; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd,copy --variants $V --iters 30; done > gpurun_out/sweep36.jsonl 2> gpurun_out/sweep36.err
cat gpurun_out/sweep36.jsonl
