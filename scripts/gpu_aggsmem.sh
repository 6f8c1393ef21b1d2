set -x
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 600 python -m pytest tests/test_gpu_aggregate.py -x -q > gpurun_out/pytest_agg.log 2>&1; echo "agg exit $?"
timeout 300 python scripts/agg_probe.py 2 20 > gpurun_out/agg_probe_smem.txt 2>&1; echo "probe exit $?"
FMMT_AGG_STAGED=0 timeout 300 python scripts/agg_probe.py 2 20 > gpurun_out/agg_probe_warp.txt 2>&1; echo "probe0 exit $?"
