set -x
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_aggregate.py -x -q > gpurun_out/pytest_agg.log 2>&1; echo "agg exit $?"
timeout 300 python scripts/agg_probe.py 2 20 > gpurun_out/agg_probe.txt 2>&1; echo "probe exit $?"
timeout 600 ncu --set full --clock-control none --import-source on -k regex:'k_aggregate|k_disaggregate_partial' -s 3 -c 4 -o gpurun_out/prof_agg2 python scripts/agg_probe.py 2 1 > gpurun_out/ncu_agg.log 2>&1; echo "ncu exit $?"
