set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_parity.py -q -x -k "fullsize or shapes or single" > gpurun_out/pytest_z64.log 2>&1; echo "z64 exit $?"
for c in 4 5; do
  timeout 900 python bench.py --config $c --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg$c.log 2>&1; echo "cfg $c exit $?"
done
