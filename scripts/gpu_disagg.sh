set -x
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_aggregate.py -x -q > gpurun_out/pytest_agg.log 2>&1; echo "agg exit $?"
timeout 300 python scripts/agg_probe.py 2 20 > gpurun_out/agg_probe_smem2.txt 2>&1; echo "probe exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_agg_v16.log 2>&1; echo "bench exit $?"
