set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_tcgemm.py -x -q > gpurun_out/pytest_tc.log 2>&1; echo "tc exit $?"
for g in tc tc1 ffma; do
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gemm $g > gpurun_out/bench_$g.log 2>&1; echo "bench $g exit $?"
done
FMMT_GRAPHS=0 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gemm tc > gpurun_out/bench_tc_nographs.log 2>&1; echo "bench nographs exit $?"
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu exit $?"
