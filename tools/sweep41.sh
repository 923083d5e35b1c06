#!/bin/bash
# end-zone pipeline depth (LMBP_EW_END_DEPTH / _MULT): shallow rings for the last tiles
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_*.so; do n=$(basename $f .so); n=${n#liblmbp_}; V="$V ${n%%-*}:@$f"; done
for c in c4 c2 c5 c3; do timeout 900 python tools/sweep.py --config $c --kernels act_fwd,act_bwd --variants $V --iters 40; done > gpurun_out/sweep41.jsonl 2> gpurun_out/sweep41.err
