#!/bin/bash
# default bench line (C4, every section) + the stream/graph keys for every BASELINE config
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/stream_all
timeout 900 python bench.py > gpurun_out/stream_all/bench_default.log 2>&1; echo "rc=$?" >> gpurun_out/stream_all/bench_default.log
for cfg in ${CONFIGS:-c1 c2 c3 c5}; do
  timeout 300 python bench.py --config $cfg --no-strong --no-fitter --no-cpu-baseline --e2e-steps 0 > gpurun_out/stream_all/bench_$cfg.log 2>&1
done
for f in gpurun_out/stream_all/bench_*.log; do
python - $f <<'PY'
import json,sys
l=[x for x in open(sys.argv[1]) if x.startswith("{")]
if not l: print(sys.argv[1], "NO LINE", open(sys.argv[1]).read()[-1500:]); sys.exit()
d=json.loads(l[-1]); s=d["stream"]; g=s["graph"]
print(json.dumps({"f":sys.argv[1].split("/")[-1],"iso":d["value"],"iso_frac":d["fraction_of_measured_peak"],"stream":s["value"],"stream_frac":s["fraction_of_measured_peak"],
 "host_ms":s["host_enqueue_ms_per_step"],"stream_ms":s["ms_per_step"],"graph":g["value"],"graph_frac":g["fraction_of_measured_peak"],"graph_ms":g["ms_per_step"],
 "s_us":{k:v["us"] for k,v in s["kernels"].items()},"g_us":{k:v["us"] for k,v in g["kernels"].items()},"iso_us":{k:v["us"] for k,v in d["kernels"].items()}}))
PY
done
