set -x
cd $GRAFT_REPO_ROOT
export FMMT_WS=1
PYTHONPATH=. timeout 120 python scripts/z64_debug.py 16 16 16 41 > gpurun_out/ws_dbg.log 2>&1; echo "dbg exit $?"
timeout 300 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc_ws.log 2>&1; echo "tc exit $?"
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multicomp.py -x -q > gpurun_out/pytest_gpu_ws.log 2>&1; echo "gpu exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ws.log 2>&1; echo "bench exit $?"
