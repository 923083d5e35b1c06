cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c4 c5 c2 c3; do timeout 600 python tools/sweep.py --config $c --kernels copy,act_fwd,act_bwd,norm_fwd,norm_bwd --variants cur: --iters 40; done > gpurun_out/sweep4.jsonl 2> gpurun_out/sweep4.err
