#!/bin/bash
# full GPU suite (incl. the exhaustive 16-bit parity) + the default bench line
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -rf > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_exhaustive16.py -m gpu -q -p no:cacheprovider -s -k act_fwd > gpurun_out/exhaustive16.log 2>&1
[ -z "$SKIP_BENCH" ] && timeout 900 python bench.py ${BENCH_ARGS} > gpurun_out/bench.log 2>&1
tail -5 gpurun_out/pytest_gpu.log; grep "not correctly" gpurun_out/exhaustive16.log | grep -v 'print(f' | cut -c1-400; tail -c 600 gpurun_out/bench.log; true
