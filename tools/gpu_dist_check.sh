#!/bin/bash
cd "${GRAFT_REPO_ROOT:-/root/repo}"
OUT=gpurun_out
( time python bench.py ) > $OUT/bench_default.log 2>&1
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29511 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-cpu-baseline > $OUT/bench_n2_gloo.log 2>&1; echo "rc=$?" >> $OUT/bench_n2_gloo.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 1 --master-addr 127.0.0.1 --master-port 29512 bench.py --gpus 1 --steps 5 --warmup 3 --no-cpu-baseline > $OUT/bench_n1_torchrun.log 2>&1; echo "rc=$?" >> $OUT/bench_n1_torchrun.log
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29513 bench.py --impl reference --gpus 2 --steps 3 --warmup 1 > $OUT/bench_ref_n2.log 2>&1; echo "rc=$?" >> $OUT/bench_ref_n2.log
( time python bench.py --impl reference ) > $OUT/bench_ref_default.log 2>&1
