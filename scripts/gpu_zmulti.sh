set -x
cd $GRAFT_REPO_ROOT
FMMT_ZMULTI=1 timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --formats tt4d@1e-04,tt4d@1e-06 > gpurun_out/bench_zm1.log 2>&1; echo "zm1 exit $?"
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --formats tt4d@1e-04,tt4d@1e-06 > gpurun_out/bench_zm0.log 2>&1; echo "zm0 exit $?"
