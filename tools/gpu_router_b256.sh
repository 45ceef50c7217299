# base-256 INT8 router: mixed-signedness probe, router tests, A/B bench against the base-128 build
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 60 ./tools/probes/i8_sign_probe > gpurun_out/i8_sign_probe.log 2>&1; echo "probe rc=$?" >> gpurun_out/i8_sign_probe.log
timeout 900 python -m pytest tests/test_gpu_router_i8.py tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/b256_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/b256_tests.log
for v in default b128; do
  if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
  for rep in 1 2; do
    NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 --no-train > gpurun_out/b256_${v}_$rep.json 2>&1
    python - <<PY
import json
j = json.loads(open("gpurun_out/b256_${v}_$rep.json").read().strip().splitlines()[-1])
s = j["stages"]
print("$v rep $rep: step %.4f ms route %.1f router %.1f select+gates %.1f gemm1 %.1f" % (
    j["ms_per_step"], s["route_ms"] * 1e3, s["router_scores_ms"] * 1e3, s["select_gates_ms"] * 1e3, s["gemm1_ms"] * 1e3))
PY
  done
done
