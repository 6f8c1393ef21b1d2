#!/bin/bash
# GPU session: warp-specialised packed pipeline (producer warp, MMA warp, 4 drain/epilogue warps) and
# producer-side fused packs; tests, bench configs 2 and 5, A/B without the fused packs.
cd "$GRAFT_REPO_ROOT"
timeout 600 python -m pytest tests/test_gpu_tcgemm.py tests/test_gpu_parity.py tests/test_gpu_realops.py -m "gpu and not slow" -x -q > gpurun_out/pytest_e.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_e.log
cp gpurun_out/parity_errors.json gpurun_out/parity_errors_e.json 2>/dev/null
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_e.json 2> gpurun_out/bench_c2_e.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_e.json 2> gpurun_out/bench_c5_e.err; echo "bench c5 rc=$?"
FMMT_FUSE_PACK=0 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_e_nofuse.json 2> gpurun_out/bench_c5_e_nofuse.err; echo "bench c5 nofuse rc=$?"
