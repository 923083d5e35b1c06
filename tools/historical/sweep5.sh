cd "${GRAFT_REPO_ROOT:-/root/repo}"
V="cur: nocodes:LMBP_DIAG_NO_CODES nomath:LMBP_DIAG_NO_MATH nomathnocodes:LMBP_DIAG_NO_MATH,LMBP_DIAG_NO_CODES w20u2s3:LMBP_FWD_W=20,LMBP_FWD_U=2,LMBP_FWD_S=3 w24u1s4:LMBP_FWD_W=24,LMBP_FWD_U=1,LMBP_FWD_S=4 w8u2s4:LMBP_FWD_W=8,LMBP_FWD_U=2,LMBP_FWD_S=4"
for c in c5 c4; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd --variants $V --iters 30; done > gpurun_out/sweep5.jsonl 2> gpurun_out/sweep5.err
