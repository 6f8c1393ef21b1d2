set -x
cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests/test_gpu_packed_paths.py -x -q > gpurun_out/pytest_packed.log 2>&1; echo "packed exit $?"
