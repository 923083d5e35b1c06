#!/bin/bash
# ncu --set full of the k = 4 SiLU step forward / backward at C4 (tools/step4_prof_driver.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:ew_tma -c 2 -o gpurun_out/prof_step4 python tools/step4_prof_driver.py > gpurun_out/ncu_step4.log 2>&1; echo "ncu rc=$?" >> gpurun_out/ncu_step4.log
tail -3 gpurun_out/ncu_step4.log; ls -la gpurun_out
