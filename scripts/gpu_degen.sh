set -x
cd $GRAFT_REPO_ROOT
timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "degenerate" > gpurun_out/pytest_degen.log 2>&1; echo "degen exit $?"
