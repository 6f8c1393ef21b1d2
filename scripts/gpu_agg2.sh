set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_aggregate.py -x -q > gpurun_out/pytest_agg.log 2>&1; echo "agg exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_agg2.log 2>&1; echo "bench exit $?"
