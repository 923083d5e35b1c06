cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd --variants nr: mufu:LMBP_SILU_MUFU_RCP; done > gpurun_out/sweep3.jsonl 2> gpurun_out/sweep3.err
