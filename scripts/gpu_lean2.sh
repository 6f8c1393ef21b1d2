set -x
cd $GRAFT_REPO_ROOT
export FMMT_WS=1
timeout 300 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc_ws.log 2>&1; echo "tcws exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "translate or restore" > gpurun_out/pytest_par_ws.log 2>&1; echo "parws exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lean2_ws.log 2>&1; echo "benchws exit $?"
unset FMMT_WS
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_lean2.log 2>&1; echo "bench exit $?"
