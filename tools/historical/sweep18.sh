cd "${GRAFT_REPO_ROOT:-/root/repo}"
V="cur: old:@paper_2406_16282_b200/_variants/liblmbp_old.so"
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd,norm_fwd,norm_bwd --variants $V --iters 20; done > gpurun_out/sweep18.jsonl 2> gpurun_out/sweep18.err
timeout 900 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/pytest_gpu.log
timeout 600 python bench.py > gpurun_out/bench_c4.log 2>&1
