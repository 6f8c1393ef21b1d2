set -x
cd $GRAFT_REPO_ROOT
CMD="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:'k_(tc_|conv_z|fwd_xy|inv_xy|cgemm|dirsum)' --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 exit $?"
C2="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-06"
timeout 300 $C2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_conv_z' -s 2 -c 1 -o gpurun_out/prof_z_tt4d $C2 > gpurun_out/ncu_full1.log 2>&1; echo "ncu2 exit $?"
C3="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats htucker4d@1e-06"
timeout 300 $C3 > gpurun_out/plain3.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_cgemm' -s 4 -c 2 -o gpurun_out/prof_cgemm_ht $C3 > gpurun_out/ncu_full2.log 2>&1; echo "ncu3 exit $?"
