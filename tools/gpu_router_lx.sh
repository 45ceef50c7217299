# INT8 router x-digit count A/B: tests of the LX=3 build, bench lines, traces
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/libnimg_moe_lx3.so timeout 900 python -m pytest tests/test_gpu_router_i8.py tests/test_gpu_parity.py \
  -m gpu -q -x -p no:cacheprovider > gpurun_out/lx3_tests.log 2>&1
echo "lx3 tests rc=$? $(tail -1 gpurun_out/lx3_tests.log)"
timeout 900 python -m pytest tests/test_gpu_router_i8.py -m gpu -q -x -p no:cacheprovider > gpurun_out/lx4_tests.log 2>&1
echo "lx4 tests rc=$? $(tail -1 gpurun_out/lx4_tests.log)"
for v in default lx3 default lx3; do
  if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
  NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 --no-train > gpurun_out/lx_$v.json 2>&1
  python - <<PY
import json
j = json.loads(open("gpurun_out/lx_$v.json").read().strip().splitlines()[-1])
s = j["stages"]
print("$v: step %.4f ms route %.1f router %.1f select+gates %.1f gemm1 %.1f" % (
    j["ms_per_step"], s["route_ms"] * 1e3, s["router_scores_ms"] * 1e3, s["select_gates_ms"] * 1e3, s["gemm1_ms"] * 1e3))
PY
done
for v in trace lx3_trace; do
  echo "== $v"
  N=3 NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/libnimg_moe_$v.so timeout 300 python tools/router_variants.py 2>&1 | tail -3
done
