#!/bin/bash
# profile pass: parity (quick), bench, filtered ncu launch list, ncu --set full of each lmbp kernel
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
OUT=gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $OUT/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> $OUT/pytest_gpu.log
for cfg in ${BENCH_CFGS:-c4}; do
  timeout 600 python bench.py --config $cfg --steps 100 --warmup 10 ${BENCH_EXTRA} > $OUT/bench_$cfg.log 2>&1; echo "bench rc=$?" >> $OUT/bench_$cfg.log
done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ew_tma|norm_" -c 40 --csv --log-file $OUT/launches.csv python bench.py --steps 5 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_launch.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch.log
if [ -n "${FULL}" ]; then
  timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ew_tma|norm_" -s 8 -c 4 -o $OUT/prof_c4 python bench.py --steps 3 --warmup 2 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_full.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full.log
fi
tail -2 $OUT/pytest_gpu.log $OUT/ncu_launch.log
