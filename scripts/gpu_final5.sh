set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "gpu exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_final5.log 2>&1; echo "bench exit $?"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg4_final.log 2>&1; echo "b4 exit $?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg5_final.log 2>&1; echo "b5 exit $?"
