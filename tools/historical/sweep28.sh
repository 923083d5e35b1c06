cd "${GRAFT_REPO_ROOT:-/root/repo}"
# (historical: the LMBP_FMA_RCP_PAIRS knob was removed after this sweep; see DESIGN 5.3)
mkdir -p gpurun_out
timeout 900 python tools/sweep.py --config c4 --kernels act_fwd,copy --iters 40 --variants base:@paper_2406_16282_b200/liblmbp.so r1:LMBP_FMA_RCP_PAIRS=1 r2:LMBP_FMA_RCP_PAIRS=2 r4:LMBP_FMA_RCP_PAIRS=4 base2:@paper_2406_16282_b200/liblmbp.so > gpurun_out/sweep_rcp.jsonl 2> gpurun_out/sweep_rcp.err
cat gpurun_out/sweep_rcp.jsonl; tail -3 gpurun_out/sweep_rcp.err
