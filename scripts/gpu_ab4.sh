set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "gpu exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --gemm tc > gpurun_out/bench_tc.log 2>&1; echo "bench exit $?"
CMD="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tucker3d@1e-06,tt4d@1e-06"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_fwd_xy|k_tc_conv_z' -s 4 -c 4 -o gpurun_out/prof_xyz $CMD > gpurun_out/ncu_full.log 2>&1; echo "ncu exit $?"
