#!/bin/bash
# ncu evidence for one config: launch list (device time + DRAM bytes per launch) and --set full of one step
cd "${GRAFT_REPO_ROOT:-/root/repo}"
CFG=${CFG:-c4}
OUT=gpurun_out
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"ew_tma|norm_" -c 40 --csv --log-file $OUT/launches_$CFG.csv python bench.py --config $CFG --steps 5 --warmup 5 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_launch_$CFG.log 2>&1; echo "ncu rc=$?" >> $OUT/ncu_launch_$CFG.log
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"ew_tma|norm_" -s 12 -c 4 -o $OUT/prof_$CFG python bench.py --config $CFG --steps 3 --warmup 3 --no-cpu-baseline --e2e-steps 0 > $OUT/ncu_full_$CFG.log 2>&1; echo "ncu full rc=$?" >> $OUT/ncu_full_$CFG.log
for ch in "8 2" "16 2" "16 3" "32 3" "64 4"; do set -- $ch; timeout 300 python bench.py --config $CFG --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 10 --e2e-chunks $1 --e2e-streams $2 | python -c "import json,sys; d=json.loads(sys.stdin.readlines()[-1]); print('$1 $2', d['e2e'])" >> $OUT/e2e_sweep_$CFG.txt 2>&1; done
