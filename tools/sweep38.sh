#!/bin/bash
# one CTA per SM with more warps / stages (uniform per-CTA rates -> short pipeline drain) vs two CTAs per SM
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_*.so; do n=$(basename $f .so); n=${n#liblmbp_}; case $n in trace*) continue;; esac; V="$V ${n%%-*}:@$f"; done
for c in c2 c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd --variants $V --iters 30; done > gpurun_out/sweep38.jsonl 2> gpurun_out/sweep38.err
cat gpurun_out/sweep38.jsonl
