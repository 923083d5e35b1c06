#!/bin/bash
# ncu --set full of the kernels of one bench config (one step), summary in gpurun_out
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=${CFG:-c2}
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ew_tma|norm_" -s 12 -c 4 -o gpurun_out/prof_$CFG python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_full_$CFG.log 2>&1; echo "rc=$?" >> gpurun_out/ncu_full_$CFG.log
