#!/bin/bash
# One GPU validation pass (run under gpurun): the -m gpu suite, smoke(), the default bench line (config 5 +
# extra configs), and the ncu launch list of the same command.  Usage: scripts/gpu_check.sh TAG [pytest-args]
# Outputs land in gpurun_out/TAG_*.
TAG=${1:-check}; shift
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,temperature.gpu --format=csv > gpurun_out/${TAG}_smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q ${@} > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests rc=$?"
tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1200 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"
cat gpurun_out/${TAG}_bench.json | head -c 600; echo
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/${TAG}_launches.csv python bench.py --quick --steps 2 --warmup 3 --no-extra \
  > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu launches rc=$?"
