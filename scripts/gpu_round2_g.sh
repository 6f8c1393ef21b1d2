#!/bin/bash
# GPU session: batch-size A/B at config 5 (Tucker-3D chain), config 2 check.
cd "$GRAFT_REPO_ROOT"
for mb in 96 256 512 1024; do
  FMMT_BATCH_MB=$mb timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --formats tucker3d@0.0001 > gpurun_out/bench_c5_g_$mb.json 2> gpurun_out/bench_c5_g_$mb.err; echo "c5 $mb rc=$?"
done
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_g.json 2> gpurun_out/bench_c2_g.err; echo "bench c2 rc=$?"
