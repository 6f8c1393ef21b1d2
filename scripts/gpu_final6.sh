set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_packed_paths.py -x -q > gpurun_out/pytest_final6.log 2>&1; echo "par exit $?"
for r in 1 2; do timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_f6_$r.log 2>&1; echo "b$r exit $?"; done
