set -x
cd $GRAFT_REPO_ROOT
CMD="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline"
timeout 600 $CMD > gpurun_out/plain.log 2>&1 && \
timeout 1200 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_(tc_|conv_z|fwd_xy|inv_xy|cgemm|dirsum)' --csv --log-file gpurun_out/launches.csv $CMD > gpurun_out/ncu_launch.log 2>&1; echo "ncu1 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_conv_z' -s 8 -c 2 -o gpurun_out/prof_tc_conv_z $CMD > gpurun_out/ncu_full1.log 2>&1; echo "ncu2 exit $?"
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_cgemm' -s 30 -c 3 -o gpurun_out/prof_tc_cgemm $CMD > gpurun_out/ncu_full2.log 2>&1; echo "ncu3 exit $?"
