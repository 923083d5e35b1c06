cd "${GRAFT_REPO_ROOT:-/root/repo}"
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider -k norm > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels norm_bwd --variants new: --iters 20; done > gpurun_out/sweep14.jsonl 2> gpurun_out/sweep14.err
