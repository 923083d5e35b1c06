#!/bin/bash
# the default bench 5x on one lease: median and spread of the C4 headline (DESIGN 5.3)
cd "${GRAFT_REPO_ROOT:-/root/repo}"
for i in 1 2 3 4 5; do
  s=$(date +%s.%N); timeout 900 python bench.py > gpurun_out/bench5_$i.log 2>&1; e=$(date +%s.%N)
  echo "run $i rc=$? wall_s=$(python -c "print(round($e-$s,1))")" >> gpurun_out/bench5_wall.txt
done
python - <<'PY'
import json, statistics
vals = []
for i in range(1, 6):
    L = [l for l in open(f"gpurun_out/bench5_{i}.log") if l.startswith("{")]
    d = json.loads(L[-1]); vals.append(d)
v = [d["value"] for d in vals]
print(json.dumps({"runs": v, "median": statistics.median(v), "min": min(v), "max": max(v),
                  "act_fwd_us": [d["kernels"]["act_fwd"]["us"] for d in vals],
                  "frac": [d["roofline"]["frac"] for d in vals],
                  "e2e": [d["e2e"]["value"] for d in vals], "clocks": [d["clocks"]["sm_mhz"] for d in vals],
                  "stream": [d["stream"]["value"] for d in vals],
                  "graph": [d["stream"]["graph"]["value"] for d in vals],
                  "graph_act_fwd_frac": [d["stream"]["graph"]["kernels"]["act_fwd"]["frac"] for d in vals]}))
PY
cat gpurun_out/bench5_wall.txt
