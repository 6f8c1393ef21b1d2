set -x
cd $GRAFT_REPO_ROOT
C2="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tucker3d@1e-06"
timeout 300 $C2 > gpurun_out/plain_m2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_cgemm' -s 7 -c 1 -o gpurun_out/prof_mode2 $C2 > gpurun_out/ncu_m2.log 2>&1; echo "ncu exit $?"
