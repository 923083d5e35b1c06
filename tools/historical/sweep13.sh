cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels norm_bwd --variants cur: notma:LMBP_NORM_NO_TMA --iters 20; done > gpurun_out/sweep13.jsonl 2> gpurun_out/sweep13.err
