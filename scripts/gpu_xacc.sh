set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "tc exit $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_d3.log 2>&1; echo "bench exit $?"
