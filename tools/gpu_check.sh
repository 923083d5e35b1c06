#!/bin/bash
# parity pass + one bench: pytest -m gpu (all, no -x), bench at C4, smoke
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1200 python -m pytest ${PYTEST_SEL:-tests} -m gpu -q -p no:cacheprovider --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
tail -3 $OUT/smoke.log; tail -25 $OUT/pytest_gpu.log; tail -c 3000 $OUT/bench.log
