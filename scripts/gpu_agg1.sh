set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_aggregate.py -x -q > gpurun_out/pytest_agg.log 2>&1; echo "agg exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multicomp.py -x -q > gpurun_out/pytest_par.log 2>&1; echo "par exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_agg.log 2>&1; echo "bench exit $?"
timeout 600 python scripts/table2_sweep.py --gamma 1e-5 32 64 > gpurun_out/table2_sweep_g1e-5.jsonl 2> gpurun_out/table2_sweep_g1e-5.err; echo "sweep exit $?"
