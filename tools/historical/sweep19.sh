cd "${GRAFT_REPO_ROOT:-/root/repo}"
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels norm_bwd --variants b224: b200:LMBP_NORM_SMEM_KB=200 b160:LMBP_NORM_SMEM_KB=160 --iters 30; done > gpurun_out/sweep19.jsonl 2> gpurun_out/sweep19.err
