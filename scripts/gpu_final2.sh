set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python scripts/table2_sweep.py 32 64 128 > gpurun_out/table2_sweep.jsonl 2> gpurun_out/table2_sweep.err; echo "sweep exit $?"
C0="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $C0 > gpurun_out/plain0.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_(tc_|conv_z|fwd_xy|inv_xy|cgemm|dirsum)' --csv --log-file gpurun_out/launches_v7.csv $C0 > gpurun_out/ncu_l.log 2>&1; echo "ncu0 exit $?"
C2="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-06"
timeout 300 $C2 > gpurun_out/plain2.log 2>&1 && \
timeout 900 ncu --set full --clock-control none --import-source on -k regex:'k_tc_conv_z' -s 1 -c 1 -o gpurun_out/prof_z_tt4d_v7 $C2 > gpurun_out/ncu_tt4d.log 2>&1; echo "ncu2 exit $?"
