#!/bin/bash
# PDL A/B: GPU suite with PDL on, then the bench (stream key) with LMBP_PDL=0 / 1 at C4 and C2
cd "${GRAFT_REPO_ROOT:-/root/repo}"
mkdir -p gpurun_out/pdl
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pdl/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pdl/pytest_gpu.log
tail -2 gpurun_out/pdl/pytest_gpu.log
for cfg in c4 c2; do
  for pdl in 0 1; do
    LMBP_PDL=$pdl timeout 300 python bench.py --config $cfg --no-strong --no-fitter --no-cpu-baseline --e2e-steps 0 \
      > gpurun_out/pdl/bench_${cfg}_pdl${pdl}.log 2>&1
    python - $cfg $pdl <<'PY'
import json,sys
l=[x for x in open(f"gpurun_out/pdl/bench_{sys.argv[1]}_pdl{sys.argv[2]}.log") if x.startswith("{")]
if not l: print(sys.argv[1:], "NO LINE"); sys.exit()
d=json.loads(l[-1]); s=d["stream"]
print(sys.argv[1:], "isolated", d["value"], d["ms_per_step"], "stream", s["value"], s["ms_per_step"], s["fraction_of_measured_peak"],
      {k:(v["us"],v["frac"]) for k,v in s["kernels"].items()}, {k:v["us"] for k,v in d["kernels"].items()})
PY
  done
done
