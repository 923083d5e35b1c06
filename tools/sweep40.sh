#!/bin/bash
# k-bit forwards: per-CTA code table (k >= 3, 16-bit) vs the compare / mux tree (LMBP_NO_CTAB)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_*.so; do n=$(basename $f .so); n=${n#liblmbp_}; V="$V ${n%%-*}:@$f"; done
for c in c4 c2 c5; do timeout 900 python tools/sweep.py --config $c --kernels step3_fwd,step4_fwd,step2_fwd --variants $V --iters 30; done > gpurun_out/sweep40.jsonl 2> gpurun_out/sweep40.err
cat gpurun_out/sweep40.jsonl
