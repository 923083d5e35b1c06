#!/bin/bash
# pipeline depth of the SiLU forward, the fused ReSwiGLU2 pair and the norm row pipeline
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_*.so; do n=$(basename $f .so); n=${n#liblmbp_}; V="$V ${n%%-*}:@$f"; done
for c in c4 c5 c2; do timeout 900 python tools/sweep.py --config $c --kernels act_fwd,swiglu_fwd,swiglu_bwd,norm_bwd --variants $V --iters 30; done > gpurun_out/sweep39.jsonl 2> gpurun_out/sweep39.err
cat gpurun_out/sweep39.jsonl
