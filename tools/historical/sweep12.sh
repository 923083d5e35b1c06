cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c4 c5 c3 c2; do timeout 600 python tools/sweep.py --config $c --kernels norm_fwd,norm_bwd --variants cur: full:LMBP_NORM_FULL_GRID rpw1:LMBP_NORM_RPW=1 rpw2:LMBP_NORM_RPW=2 rpw4:LMBP_NORM_RPW=4 rpw8:LMBP_NORM_RPW=8 --iters 20; done > gpurun_out/sweep12.jsonl 2> gpurun_out/sweep12.err
