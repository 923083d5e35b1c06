#!/bin/bash
# bench (default config) + ncu of the fitter kernels + refreshed C4 launch list / full profile
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out; mkdir -p $OUT
timeout 900 python bench.py > $OUT/bench_full.log 2>&1; echo "bench rc=$?" >> $OUT/bench_full.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"fit_" -c 8 -o $OUT/prof_fit python tools/fit_prof_driver.py > $OUT/ncu_fit.log 2>&1; echo "ncu fit rc=$?" >> $OUT/ncu_fit.log
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ew_tma|norm_" -c 40 --csv --log-file $OUT/launches_c4.csv python bench.py --steps 5 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-fitter > $OUT/ncu_launch_c4.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch_c4.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ew_tma|norm_" -s 12 -c 4 -o $OUT/prof_c4 python bench.py --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-fitter > $OUT/ncu_full_c4.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full_c4.log
tail -2 $OUT/*.log
