cd "${GRAFT_REPO_ROOT:-/root/repo}"
V="base: s3:LMBP_TMA_STAGES=3 s6:LMBP_TMA_STAGES=6 u2:LMBP_TMA_U=2 u8s3:LMBP_TMA_U=8,LMBP_TMA_STAGES=3 w4:LMBP_TMA_WARPS=4 w12:LMBP_TMA_WARPS=12,LMBP_TMA_STAGES=3 nef:LMBP_NO_EVICT_FIRST cs:LMBP_ST_CS"
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd --variants $V; done > gpurun_out/sweep1.jsonl 2> gpurun_out/sweep1.err
