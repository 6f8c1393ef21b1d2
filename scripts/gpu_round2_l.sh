#!/bin/bash
# GPU session: all-64-kz z-stage tiles (BN = 64, two epilogue warpgroups); parity, bench; memory-bounded
# TT-SVD / Gram paths at 256^3 x 435 (probe + sweeps).
cd "$GRAFT_REPO_ROOT"
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_l.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/pytest_l.log
timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/bench_c5_l.json 2> gpurun_out/bench_c5_l.err; echo "bench c5 rc=$?"
timeout 600 python scripts/mem_probe.py tucker3d tucker4d tt4d > gpurun_out/mem_probe_l.log 2>&1; echo "probe rc=$?"
