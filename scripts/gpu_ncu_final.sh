set -x
cd $GRAFT_REPO_ROOT
C0="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline"
timeout 300 $C0 > gpurun_out/plain_final.log 2>&1 && \
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_(tc_|conv_z|fwd_xy|inv_xy|cgemm|dirsum|aggregate|disaggregate)' --csv --log-file gpurun_out/launches_final.csv $C0 > gpurun_out/ncu_lf.log 2>&1; echo "ncu exit $?"
