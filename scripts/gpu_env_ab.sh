#!/bin/bash
# A/B of one runtime switch (run under gpurun): scripts/gpu_env_ab.sh TAG VAR val1 val2 ... [-- pytest-k-expression]
TAG=$1; VAR=$2; shift 2
VALS=()
while [ $# -gt 0 ] && [ "$1" != "--" ]; do VALS+=("$1"); shift; done
[ "$1" = "--" ] && shift
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
if [ $# -gt 0 ]; then
  timeout 1200 python -m pytest tests -m "gpu and not slow" -q -k "$1" > gpurun_out/${TAG}_targeted.log 2>&1; echo "targeted rc=$?"
  tail -4 gpurun_out/${TAG}_targeted.log
fi
for v in "${VALS[@]}"; do
  env $VAR=$v timeout 600 python bench.py --no-extra --no-cpu-baseline --steps 5 --warmup 3 \
    > gpurun_out/${TAG}_bench_${VAR}${v}.json 2> gpurun_out/${TAG}_bench_${VAR}${v}.err; echo "bench $VAR=$v rc=$?"
  python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench_${VAR}${v}.json").read().strip().splitlines()[-1])
print("$VAR=$v", d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "dense", d["dense"]["ms"],
      {k: x["ms_per_launch"] for k, x in d["kernels"].items()})
PY
done
