set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "tc exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_par.log 2>&1; echo "par exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_late.log 2>&1; echo "bench exit $?"
