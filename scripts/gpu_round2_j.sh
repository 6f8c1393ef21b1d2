#!/bin/bash
# GPU session: chunked four-step xy FFT (2 CTAs / SM at 128^2 planes); tests + bench configs 2, 4, 5.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_j.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_j.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_j.json 2> gpurun_out/bench_c2_j.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_j.json 2> gpurun_out/bench_c5_j.err; echo "bench c5 rc=$?"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c4_j.json 2> gpurun_out/bench_c4_j.err; echo "bench c4 rc=$?"
