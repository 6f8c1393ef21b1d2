set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tucker3d" > gpurun_out/pytest_m2b.log 2>&1; echo "par exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_m2b.log 2>&1; echo "bench exit $?"
