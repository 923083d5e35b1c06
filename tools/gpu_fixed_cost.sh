#!/bin/bash
# fixed-cost decomposition of the activation kernels across variants (tools/probes/fixed_cost.py),
# then CTA timelines of the trace variants (tools/trace_ew.py)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
V=""; TV=""
for f in paper_2406_16282_b200/_variants/liblmbp_*.so; do n=$(basename $f .so); n=${n#liblmbp_}; n=${n%%-*}
  case $n in trace*) TV="$TV $n:@$f";; *) V="$V $n:@$f";; esac; done
timeout 900 python tools/probes/fixed_cost.py --variants $V ${FC_ARGS} > gpurun_out/fixed_cost.jsonl 2> gpurun_out/fixed_cost.err
[ -n "$TV" ] && timeout 600 python tools/trace_ew.py --variants $TV --configs ${TRACE_CONFIGS:-c4} > gpurun_out/trace.jsonl 2> gpurun_out/trace.err
grep fit gpurun_out/fixed_cost.jsonl; tail -3 gpurun_out/fixed_cost.err; cat gpurun_out/trace.jsonl; tail -3 gpurun_out/trace.err
