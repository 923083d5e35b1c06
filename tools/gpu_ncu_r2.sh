#!/bin/bash
# round-2 ncu evidence: per-config launch list of the bench step (device time + DRAM bytes per launch,
# the contract's --metrics gpu__time_duration.sum --clock-control none pass) and --set full of one step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
for CFG in ${CFGS:-c4 c2}; do
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ew_tma|norm_" -c 40 --csv --log-file $OUT/launches_$CFG.csv python bench.py --config $CFG --steps 5 --warmup 5 --no-cpu-baseline --e2e-steps 0 --no-strong --no-fitter > $OUT/ncu_launch_$CFG.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch_$CFG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ew_tma|norm_" -s 12 -c 4 -o $OUT/prof_$CFG python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 --no-strong --no-fitter > $OUT/ncu_full_$CFG.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full_$CFG.log
done
ls -la $OUT
