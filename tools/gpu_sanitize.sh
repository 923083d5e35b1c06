#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for tool in memcheck racecheck synccheck initcheck; do
  timeout 1200 compute-sanitizer --tool $tool --target-processes all --print-limit 20 python tools/sanitize_driver.py > gpurun_out/sanitize_$tool.log 2>&1; echo "rc=$?" >> gpurun_out/sanitize_$tool.log; tail -3 gpurun_out/sanitize_$tool.log
done
