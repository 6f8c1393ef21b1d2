#!/bin/bash
# A/B of experimental library builds (run under gpurun): scripts/gpu_ab.sh TAG lib1 lib2 ...  ("default" = libfmmt.so)
TAG=$1; shift
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
for lib in "$@"; do
  if [ "$lib" = default ]; then unset FMMT_LIB; else export FMMT_LIB=$lib; fi
  timeout 600 python bench.py --no-extra --no-cpu-baseline --steps 5 --warmup 3 \
    > gpurun_out/${TAG}_bench_${lib}.json 2> gpurun_out/${TAG}_bench_${lib}.err; echo "bench $lib rc=$?"
  python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench_${lib}.json").read().strip().splitlines()[-1])
print("$lib", d["value"], d["ms_per_step"], "e2e", d["e2e"]["value"], "dense", d["dense"]["ms"],
      {k: v["ms_per_launch"] for k, v in d["kernels"].items()})
PY
done
