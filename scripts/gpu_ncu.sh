#!/bin/bash
# ncu --set full capture of one kernel of the config-5 (or --config N) step, under gpurun, after the same
# command ran clean without ncu.  Usage: scripts/gpu_ncu.sh TAG FMT@TOL KERNEL_REGEX [SKIP] [COUNT] [CONFIG]
# -> gpurun_out/TAG.ncu-rep, gpurun_out/TAG_{raw,details}.csv
TAG=$1; FMT=$2; RE=$3; SKIP=${4:-6}; CNT=${5:-1}; CFG=${6:-5}
cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
CMD="python bench.py --config $CFG --quick --steps 1 --warmup 3 --formats $FMT"
timeout 900 $CMD > gpurun_out/${TAG}_plain.log 2>&1 || { echo "plain run failed"; tail -5 gpurun_out/${TAG}_plain.log; exit 1; }
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:"$RE" -s $SKIP -c $CNT \
  -o gpurun_out/$TAG -f $CMD > gpurun_out/${TAG}_ncu.log 2>&1; echo "ncu $TAG rc=$?"
ncu -i gpurun_out/$TAG.ncu-rep --page raw --csv > gpurun_out/${TAG}_raw.csv 2>/dev/null
ncu -i gpurun_out/$TAG.ncu-rep --page details --csv > gpurun_out/${TAG}_details.csv 2>/dev/null
