#!/bin/bash
# GPU session: xy sub-batches (W in L2) fixed; tests + bench configs 2, 4, 5 + W budget A/B.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_i.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_i.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_i.json 2> gpurun_out/bench_c2_i.err; echo "bench c2 rc=$?"
for w in 48 16 128; do
FMMT_W_MB=$w timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_i_w$w.json 2> gpurun_out/bench_c5_i_w$w.err; echo "bench c5 w$w rc=$?"
done
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c4_i.json 2> gpurun_out/bench_c4_i.err; echo "bench c4 rc=$?"
