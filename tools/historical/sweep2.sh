cd "${GRAFT_REPO_ROOT:-/root/repo}"
V="w12nef:LMBP_TMA_WARPS=12,LMBP_TMA_STAGES=3,LMBP_NO_EVICT_FIRST w16nef:LMBP_TMA_WARPS=16,LMBP_TMA_STAGES=3,LMBP_NO_EVICT_FIRST w12u2nef:LMBP_TMA_WARPS=12,LMBP_TMA_U=2,LMBP_TMA_STAGES=4,LMBP_NO_EVICT_FIRST w16u2nef:LMBP_TMA_WARPS=16,LMBP_TMA_U=2,LMBP_TMA_STAGES=4,LMBP_NO_EVICT_FIRST w8nef:LMBP_NO_EVICT_FIRST"
for c in c4 c5 c3; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd --variants $V; done > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
timeout 600 ncu --set full --clock-control none -k regex:act_fwd -s 2 -c 1 -o gpurun_out/prof_c5_actfwd python bench.py --config c5 --steps 2 --warmup 1 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ncu_c5.log 2>&1
