set -x
cd $GRAFT_REPO_ROOT
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/smoke.log 2>&1; echo "smoke exit $?"
timeout 900 python bench.py > gpurun_out/bench_final.log 2>&1; echo "bench exit $?"
timeout 600 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/bench_ref.log 2>&1; echo "ref exit $?"
C0="python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
  -k regex:'k_(tc_|conv_z|fwd_xy|inv_xy|cgemm|dirsum|aggregate|disaggregate)' --csv --log-file gpurun_out/launches_v12.csv $C0 > gpurun_out/ncu_l12.log 2>&1; echo "ncu exit $?"
