#!/bin/bash
# In-stream A/B of library variants: bench.py (stream key) per config per variant.
#   VARIANTS="base:@paper_2406_16282_b200/liblmbp.so stcs:@paper_2406_16282_b200/_variants/..." CONFIGS="c4 c2"
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/ab
for cfg in ${CONFIGS:-c4 c2}; do
  for v in ${VARIANTS}; do
    name=${v%%:*}; lib=${v#*:@}
    for rep in ${REPS:-1}; do
    LMBP_LIBRARY=$PWD/$lib timeout 300 python bench.py --config $cfg --no-strong --no-fitter --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/ab/bench_${cfg}_${name}_${rep}.log 2>&1
    python - $cfg $name $rep <<'PY'
import json,sys
c,n,r=sys.argv[1:]
l=[x for x in open(f"gpurun_out/ab/bench_{c}_{n}_{r}.log") if x.startswith("{")]
if not l: print(c,n,"NO LINE", open(f"gpurun_out/ab/bench_{c}_{n}_{r}.log").read()[-600:]); sys.exit()
d=json.loads(l[-1]); s=d["stream"]
print(json.dumps({"cfg":c,"variant":n,"rep":r,"isolated":d["value"],"stream":s["value"],"stream_ms":s["ms_per_step"],
 "stream_us":{k:v["us"] for k,v in s["kernels"].items()},"iso_us":{k:v["us"] for k,v in d["kernels"].items()}}))
PY
    done
  done
done
