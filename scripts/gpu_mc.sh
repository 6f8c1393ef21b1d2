set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_multicomp.py -x -q > gpurun_out/pytest_mc.log 2>&1; echo "mc exit $?"
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/pytest_gpu.log 2>&1; echo "gpu exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 > gpurun_out/bench_tc.log 2>&1; echo "bench exit $?"
