set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "tt4d" > gpurun_out/pytest_packb.log 2>&1; echo "par exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_packb.log 2>&1; echo "bench exit $?"
FMMT_PACKB=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_nopackb.log 2>&1; echo "bench0 exit $?"
