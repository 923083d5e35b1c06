cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
V="cur: w20u2s3:LMBP_FWD_W=20,LMBP_FWD_U=2,LMBP_FWD_S=3 w16u2s3:LMBP_FWD_W=16,LMBP_FWD_U=2,LMBP_FWD_S=3 w16u4s3:LMBP_FWD_W=16,LMBP_FWD_U=4,LMBP_FWD_S=3 w12u2s4:LMBP_FWD_W=12,LMBP_FWD_U=2,LMBP_FWD_S=4"
for c in c5 c4 c2; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd --variants $V --iters 30; done > gpurun_out/sweep6.jsonl 2> gpurun_out/sweep6.err
