set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_lossy.py -q > gpurun_out/pytest_lossy.log 2>&1; echo "lossy exit $?"
