cd "${GRAFT_REPO_ROOT:-/root/repo}"
V="cur: old:@paper_2406_16282_b200/_variants/liblmbp_old.so w8mb4:LMBP_FWD_MINB=4,LMBP_FWD_W=8,LMBP_FWD_U=2,LMBP_FWD_S=4 cur2: old2:@paper_2406_16282_b200/_variants/liblmbp_old.so"
for c in c4 c5; do timeout 600 python tools/sweep.py --config $c --kernels act_fwd,act_bwd,norm_fwd,norm_bwd --variants $V --iters 20; done > gpurun_out/sweep17.jsonl 2> gpurun_out/sweep17.err
nvidia-smi -q | grep -A3 -i "serial\|Clocks Event\|Product Name" | head -20 > gpurun_out/gpuinfo.txt
