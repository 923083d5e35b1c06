#!/bin/bash
# run tools/trace_ew.py on every prebuilt trace variant (_variants/liblmbp_trace*.so)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
V=""
for f in paper_2406_16282_b200/_variants/liblmbp_trace*.so; do n=$(basename $f .so); n=${n#liblmbp_}; V="$V ${n%%-*}:@$f"; done
python tools/trace_ew.py --variants $V --configs ${CONFIGS:-c2,c4,c1,c5} > gpurun_out/trace_ew.jsonl 2>&1; cat gpurun_out/trace_ew.jsonl
