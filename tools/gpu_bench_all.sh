#!/bin/bash
# the bench line for every BASELINE config (C1..C5), one after another on one lease
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out
for c in c1 c2 c3 c4 c5; do
  timeout 900 python bench.py --config $c ${BENCH_ARGS} > gpurun_out/bench_$c.log 2>&1; echo "rc=$?" >> gpurun_out/bench_$c.log
done
python - <<'PY'
import json
for c in ["c1", "c2", "c3", "c4", "c5"]:
    L = [l for l in open(f"gpurun_out/bench_{c}.log") if l.startswith("{")]
    if not L:
        print(c, "no line"); continue
    d = json.loads(L[-1])
    print(c, d["value"], d["roofline"]["kernel"], d["roofline"]["frac"], {k: (v["us"], v["frac"]) for k, v in d["kernels"].items()}, d["clocks"]["sm_mhz"], d["clocks"]["reasons"])
PY
