#!/bin/bash
# round-2 check: build, smoke, selected GPU tests, C4 bench, 2-rank self-launched bench (ranks share the GPU)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
OUT=gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.build(); g.smoke()" > $OUT/smoke.log 2>&1; echo "smoke rc=$?" >> $OUT/smoke.log
timeout 1500 python -m pytest ${PYTEST_SEL:-tests} -m gpu -q -p no:cacheprovider --durations=15 > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
timeout 900 python bench.py ${BENCH_ARGS} > $OUT/bench.log 2>&1; echo "bench rc=$?" >> $OUT/bench.log
if [ -z "$SKIP_N2" ]; then
timeout 900 python bench.py --gpus 2 --steps 10 --warmup 3 --dist-backend gloo --no-fitter > $OUT/bench_n2.log 2>&1; echo "bench n2 rc=$?" >> $OUT/bench_n2.log
fi
tail -3 $OUT/smoke.log; tail -25 $OUT/pytest_gpu.log; tail -c 1500 $OUT/bench.log; [ -z "$SKIP_N2" ] && tail -c 1500 $OUT/bench_n2.log; true
