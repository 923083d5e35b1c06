cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c2 c3 c1 c4; do timeout 600 python tools/sweep.py --config $c --kernels norm_fwd,norm_bwd --variants cur: pf:LMBP_ROW_PREFETCH=1 v8:LMBP_WARP_VMAX=8 v8pf:LMBP_WARP_VMAX=8,LMBP_ROW_PREFETCH=1 v6pf:LMBP_WARP_VMAX=6,LMBP_ROW_PREFETCH=1 --iters 20; done > gpurun_out/sweep15.jsonl 2> gpurun_out/sweep15.err
