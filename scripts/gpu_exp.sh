set -x
cd $GRAFT_REPO_ROOT
PYTHONPATH=. timeout 300 python scripts/split_exp.py > gpurun_out/split_exp.log 2>&1; echo "exp exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gemm tc1 > gpurun_out/bench_tc1.log 2>&1; echo "bench exit $?"
