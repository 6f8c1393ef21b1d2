set -x
cd $GRAFT_REPO_ROOT
PYTHONPATH=. timeout 120 python scripts/z64_debug.py 4 4 32 7 > gpurun_out/z64_a.log 2>&1; echo "z64a exit $?"
PYTHONPATH=. timeout 120 python scripts/z64_debug.py 4 4 32 17 > gpurun_out/z64_b.log 2>&1; echo "z64b exit $?"
PYTHONPATH=. timeout 120 python scripts/z64_debug.py 16 16 32 41 > gpurun_out/z64_c.log 2>&1; echo "z64c exit $?"
timeout 300 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "tc exit $?"
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_tc.log 2>&1; echo "bench exit $?"
