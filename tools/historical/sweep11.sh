cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c5 c4 c3 c2 c1; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd --variants u1:LMBP_EW_UNIT=1 u2:LMBP_EW_UNIT=2 u4:LMBP_EW_UNIT=4 u8:LMBP_EW_UNIT=8 u2w20:LMBP_EW_UNIT=2,LMBP_FWD_W=20,LMBP_FWD_U=2,LMBP_FWD_S=3 --iters 20; done > gpurun_out/sweep11.jsonl 2> gpurun_out/sweep11.err
