#!/bin/bash
# GPU session: non-blocking producer in the packed pipeline; GEMM hook + parity + bench; ncu of the z-stage.
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_gpu_tcgemm.py tests/test_gpu_parity.py -x -q > gpurun_out/pytest_d.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_d.log
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_d.json 2> gpurun_out/bench_c2_d.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_d.json 2> gpurun_out/bench_c5_d.err; echo "bench c5 rc=$?"
timeout 300 python bench.py --config 2 --quick --steps 1 --warmup 3 --formats tt4d@1e-06,tucker3d@1e-06 > gpurun_out/plain_d.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"k_pk_conv_z|k_pk_cgemm" -s 6 -c 4 -o gpurun_out/prof_d python bench.py --config 2 --quick --steps 1 --warmup 3 --formats tt4d@1e-06,tucker3d@1e-06 > gpurun_out/ncu_d.log 2>&1; echo "ncu rc=$?"
