set -x
cd $GRAFT_REPO_ROOT
C2="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-06"
timeout 300 $C2 > gpurun_out/plain15.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_conv_z' -s 1 -c 1 -o gpurun_out/prof_z_tt4d_v15 $C2 > gpurun_out/ncu15.log 2>&1; echo "ncu exit $?"
