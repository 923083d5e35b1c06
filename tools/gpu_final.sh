#!/bin/bash
# What the driver runs at round end, on one box: GPU suite, smoke, the default bench, the reference arm.
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/final
timeout 1200 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/final/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/final/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/final/smoke.log
timeout 900 python bench.py --impl reference > gpurun_out/final/bench_reference.log 2>&1; echo "rc=$?" >> gpurun_out/final/bench_reference.log
timeout 900 python bench.py > gpurun_out/final/bench.log 2>&1; echo "rc=$?" >> gpurun_out/final/bench.log
tail -2 gpurun_out/final/pytest_gpu.log; tail -2 gpurun_out/final/smoke.log
grep "^{" gpurun_out/final/bench_reference.log | cut -c1-300
grep "^{" gpurun_out/final/bench.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline']['frac'], d['stream']['value'], d['e2e']['value'], d['clocks'], d['build']['matches_sources'])"
