#!/bin/bash
# GPU session: fast GPU tests, the bench (config 5 headline + configs 2, 4), then the slow real-operator tests.
cd "$GRAFT_REPO_ROOT"
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > gpurun_out/smi_a.txt 2>&1
timeout 1200 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_fast_a.log 2>&1; echo "fast tests rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_a.json 2> gpurun_out/bench_a.err; echo "bench rc=$?"
timeout 1500 python -m pytest tests -m "gpu and slow" -q > gpurun_out/pytest_slow_a.log 2>&1; echo "slow tests rc=$?"
tail -3 gpurun_out/pytest_fast_a.log gpurun_out/pytest_slow_a.log
