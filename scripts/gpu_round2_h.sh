#!/bin/bash
# GPU session: xy sub-batches (W in L2), 2 GB restore batches, 16-byte packs; tests + bench configs 2, 4, 5.
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m "gpu and not slow" -x -q > gpurun_out/pytest_h.log 2>&1; echo "tests rc=$?"
tail -2 gpurun_out/pytest_h.log
cp gpurun_out/parity_errors.json gpurun_out/parity_errors_h.json 2>/dev/null
timeout 600 python bench.py --config 2 --steps 10 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c2_h.json 2> gpurun_out/bench_c2_h.err; echo "bench c2 rc=$?"
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_h.json 2> gpurun_out/bench_c5_h.err; echo "bench c5 rc=$?"
FMMT_W_MB=16 timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_h_w16.json 2> gpurun_out/bench_c5_h_w16.err; echo "bench c5 w16 rc=$?"
timeout 900 python bench.py --config 4 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c4_h.json 2> gpurun_out/bench_c4_h.err; echo "bench c4 rc=$?"
