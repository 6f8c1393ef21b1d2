set -x
cd $GRAFT_REPO_ROOT
for v in "FMMT_NONE=1" "FMMT_ZMULTI=1" "FMMT_PACK=0" "FMMT_PACK=0 FMMT_ZMULTI=1"; do
  env $v timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline > "gpurun_out/bench_ab_${v// /_}.log" 2>&1; echo "bench [$v] exit $?"
done
