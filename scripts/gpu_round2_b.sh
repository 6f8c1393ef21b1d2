#!/bin/bash
# GPU session: the fp16-split tensor-core path (libfmmt.so) vs the TF32 split (libfmmt_tf32.so):
# accuracy (GEMM hook + restore / translate parity) and throughput at configs 2 and 5.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests/test_gpu_tcgemm.py tests/test_gpu_parity.py tests/test_gpu_parity_fullsize.py -x -q > gpurun_out/pytest_f16_b.log 2>&1; echo "f16 parity rc=$?"
cp gpurun_out/parity_errors.json gpurun_out/parity_errors_f16_b.json 2>/dev/null
for lib in f16 tf32; do
  if [ $lib = tf32 ]; then export FMMT_LIB=tf32; else unset FMMT_LIB; fi
  timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_$lib.json 2> gpurun_out/bench_c2_$lib.err; echo "bench c2 $lib rc=$?"
  timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_$lib.json 2> gpurun_out/bench_c5_$lib.err; echo "bench c5 $lib rc=$?"
done
tail -3 gpurun_out/pytest_f16_b.log
