#!/bin/bash
# GPU session: the packed-operand tensor-core pipeline (kernels_tcpk.cuh): GEMM hook, parity, then bench.
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tcgemm_c.log 2>&1; echo "tcgemm rc=$?"
tail -2 gpurun_out/pytest_tcgemm_c.log
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_fast_c.log 2>&1; echo "fast rc=$?"
tail -2 gpurun_out/pytest_fast_c.log
cp gpurun_out/parity_errors.json gpurun_out/parity_errors_c.json 2>/dev/null
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_c.json 2> gpurun_out/bench_c2_c.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_c.json 2> gpurun_out/bench_c5_c.err; echo "bench c5 rc=$?"
