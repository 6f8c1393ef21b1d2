set -x
cd $GRAFT_REPO_ROOT
timeout 120 python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-04 > gpurun_out/dbg1.log 2>&1; echo "q1 exit $?"
FMMT_GRAPHS=0 timeout 120 python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-04 > gpurun_out/dbg2.log 2>&1; echo "q2 exit $?"
timeout 120 python bench.py --quick --steps 1 --warmup 1 --no-cpu-baseline --formats tt4d@1e-06 > gpurun_out/dbg3.log 2>&1; echo "q3 exit $?"
timeout 300 python -m pytest tests/test_gpu_multicomp.py -x -q -k tt4d > gpurun_out/dbg4.log 2>&1; echo "mc exit $?"
