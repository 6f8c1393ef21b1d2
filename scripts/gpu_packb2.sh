set -x
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 90 python scripts/packb_repro.py tt4d 1e-4 2 > gpurun_out/dbg7.log 2>&1; echo "c2 exit $?"
timeout 90 python scripts/packb_repro.py tt4d 1e-6 3 > gpurun_out/dbg9.log 2>&1; echo "c3 exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multicomp.py tests/test_gpu_aggregate.py -x -q > gpurun_out/pytest_packb.log 2>&1; echo "par exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_packb.log 2>&1; echo "bench exit $?"
