#!/bin/bash
# Round-end validation under gpurun: the full -m gpu suite, smoke(), the default bench line (config 5 +
# extra configs + cpu_baseline), the reference arm, and the ncu launch list of the headline step (our kernels
# only, so setup-time library kernels are not replayed).  Usage: scripts/gpu_final.sh TAG
TAG=${1:-final}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 1800 python -m pytest tests -m gpu -q > gpurun_out/${TAG}_pytest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/${TAG}_smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python bench.py > gpurun_out/${TAG}_bench.json 2> gpurun_out/${TAG}_bench.err; echo "bench rc=$?"; head -c 400 gpurun_out/${TAG}_bench.json; echo
timeout 600 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/${TAG}_ref.json 2> gpurun_out/${TAG}_ref.err; echo "ref rc=$?"
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:"k_(pk_|tc_|tucker|fwd_|inv_|dirsum|conv_z|cgemm)" --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --quick --steps 1 --warmup 3 --no-extra > gpurun_out/${TAG}_ncu.log 2>&1; echo "launches rc=$?"
