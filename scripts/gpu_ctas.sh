set -x
cd $GRAFT_REPO_ROOT
for c in 2 3 4 6; do
FMMT_TC_CTAS=$c timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ctas$c.log 2>&1; echo "ctas$c exit $?"
done
