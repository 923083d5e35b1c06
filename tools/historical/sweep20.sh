cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k "norm or full_size" > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c4 c5 c3; do timeout 600 python tools/sweep.py --config $c --kernels norm_fwd,norm_bwd --variants rowtma: old:LMBP_NO_ROW_TMA --iters 20; done > gpurun_out/sweep20.jsonl 2> gpurun_out/sweep20.err
