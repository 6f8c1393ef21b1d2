set -x
cd $GRAFT_REPO_ROOT
for r in 1 2; do for c in 2 4; do
FMMT_TC_CTAS=$c timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench_ctasB${c}_$r.log 2>&1; echo "c$c r$r exit $?"
done; done
