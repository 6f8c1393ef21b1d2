set -x
cd $GRAFT_REPO_ROOT
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_final.log 2>&1; echo "gpu exit $?"
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_final7.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --impl reference > gpurun_out/bench_ref7.log 2>&1; echo "ref exit $?"
