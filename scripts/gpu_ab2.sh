set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "tc exit $?"
PYTHONPATH=. timeout 300 python scripts/split_exp.py > gpurun_out/split_exp.log 2>&1; echo "exp exit $?"
for g in tc tc1; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gemm $g > gpurun_out/bench_$g.log 2>&1; echo "bench $g exit $?"
done
