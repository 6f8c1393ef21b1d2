set -x
cd $GRAFT_REPO_ROOT
C1="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tucker3d@1e-06"
timeout 300 $C1 > gpurun_out/plain1.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_cgemm|k_tc_conv_z|k_fwd_xy' -s 3 -c 4 -o gpurun_out/prof_t3d $C1 > gpurun_out/ncu_t3d.log 2>&1; echo "ncu1 exit $?"
C2="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-06"
timeout 300 $C2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_conv_z' -s 1 -c 1 -o gpurun_out/prof_z_tt4d_v6 $C2 > gpurun_out/ncu_tt4d.log 2>&1; echo "ncu2 exit $?"
