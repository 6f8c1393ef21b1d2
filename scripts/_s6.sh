cd "$GRAFT_REPO_ROOT"
mkdir -p gpurun_out
timeout 900 python -m pytest -x -q tests/test_gpu_packed_paths.py -k "fused" "tests/test_gpu_parity_fullsize.py::test_config5_tucker3d_fullsize" > gpurun_out/s6_pytest.log 2>&1; echo "tests rc=$?"; tail -3 gpurun_out/s6_pytest.log
run() { tag=$1; shift; env "$@" timeout 900 python bench.py --config 5 --steps 5 --warmup 3 --no-extra --no-cpu-baseline > gpurun_out/s6_$tag.json 2> gpurun_out/s6_$tag.err; echo "bench $tag rc=$?"; tail -2 gpurun_out/s6_$tag.err; }
run c5
run c5_ns12 FMMT_ZNS=12
run c5_nocl FMMT_ZCLUSTER=0
python - <<'PY'
import json
for f in ["c5","c5_ns12","c5_nocl"]:
    try:
        d=json.loads(open(f"gpurun_out/s6_{f}.json").read().strip().splitlines()[-1])
        print(f, d["value"], d["ms_per_step"], {k:v["ms"] for k,v in d["per_format"].items()})
        print("   ", {k:(v["ms_per_launch"],v["launches"],v.get("achieved_tflops")) for k,v in list(d["kernels"].items())[:12]})
    except Exception as e: print(f, "ERR", e)
PY
