set -x
cd $GRAFT_REPO_ROOT
export PYTHONPATH=.
timeout 90 python scripts/packb_repro.py tt4d 1e-4 1 > gpurun_out/dbg6.log 2>&1; echo "c1 exit $?"
timeout 90 python scripts/packb_repro.py tt4d 1e-4 2 > gpurun_out/dbg7.log 2>&1; echo "c2 exit $?"
timeout 300 compute-sanitizer --tool racecheck --print-limit 5 python scripts/packb_repro.py tt4d 1e-4 2 > gpurun_out/dbg8.log 2>&1; echo "san exit $?"
