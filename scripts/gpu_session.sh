#!/bin/bash
# Targeted GPU check (run under gpurun) of the overlapped host upload and the single-rank NCCL path, then the
# e2e A/B (serial vs overlapped upload) at config 5.  Usage: scripts/gpu_session.sh TAG
TAG=${1:-s}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_realops.py tests/test_gpu_parity.py -m "gpu and not slow" -q \
  -k "single_rank or host_e2e or virtual_sharding" > gpurun_out/${TAG}_targeted.log 2>&1; echo "targeted rc=$?"
tail -15 gpurun_out/${TAG}_targeted.log
for ov in 1 0; do
  FMMT_H2D_OVERLAP=$ov timeout 600 python bench.py --no-extra --no-cpu-baseline --steps 5 --warmup 3 \
    > gpurun_out/${TAG}_bench_ov${ov}.json 2> gpurun_out/${TAG}_bench_ov${ov}.err; echo "bench ov=$ov rc=$?"
  python - <<PY
import json
d = json.loads(open("gpurun_out/${TAG}_bench_ov${ov}.json").read().strip().splitlines()[-1])
print("overlap=${ov}", d["value"], d["ms_per_step"], d["e2e"], d.get("dense"))
PY
done
