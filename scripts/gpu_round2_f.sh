#!/bin/bash
# GPU session: warp-specialised packed pipeline + coalesced packs; all GPU tests (fast), bench 2 and 5.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_f.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_f.log
cp gpurun_out/parity_errors.json gpurun_out/parity_errors_f.json 2>/dev/null
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_f.json 2> gpurun_out/bench_c2_f.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_f.json 2> gpurun_out/bench_c5_f.err; echo "bench c5 rc=$?"
