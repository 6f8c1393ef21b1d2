set -x
cd $GRAFT_REPO_ROOT
for c in 1 3 4 5; do
timeout 900 python bench.py --config $c --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_cfg${c}_v12.log 2>&1; echo "cfg$c exit $?"
done
