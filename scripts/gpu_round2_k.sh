#!/bin/bash
# GPU session: 2-CTA cluster multicast of the TT-4D z-stage's shared A; parity, A/B bench, ncu of the z-stages.
cd "$GRAFT_REPO_ROOT"
timeout 300 python -m pytest tests/test_gpu_parity_fullsize.py tests/test_gpu_parity.py -x -q -k "tt4d or fullsize" > gpurun_out/pytest_k.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_k.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_k.json 2> gpurun_out/bench_c5_k.err; echo "bench c5 rc=$?"
FMMT_ZCLUSTER=0 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline --formats tt4d@0.0001 > gpurun_out/bench_c5_k_nocl.json 2> gpurun_out/bench_c5_k_nocl.err; echo "bench c5 nocl rc=$?"
for f in tucker3d tt4d; do
timeout 600 python bench.py --config 5 --quick --steps 1 --warmup 3 --formats $f@0.0001 > gpurun_out/plain_k_$f.log 2>&1 && \
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:"k_pk_conv_z64" -s 6 -c 2 -o gpurun_out/prof_k_$f python bench.py --config 5 --quick --steps 1 --warmup 3 --formats $f@0.0001 > gpurun_out/ncu_k_$f.log 2>&1; echo "ncu $f rc=$?"
done
