cd "${GRAFT_REPO_ROOT:-/root/repo}"
V="w16u2s4:LMBP_FWD_W=16,LMBP_FWD_U=2,LMBP_FWD_S=4 w20u2s3:LMBP_FWD_W=20,LMBP_FWD_U=2,LMBP_FWD_S=3"
for c in c5 c4; do for off in 0 65536 1048576 2113536 33554432; do timeout 600 python tools/sweep.py --config $c --kernels copy,act_fwd,act_bwd --variants $V --iters 20 --yoff $off; done; done > gpurun_out/sweep8.jsonl 2> gpurun_out/sweep8.err
