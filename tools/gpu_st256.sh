# 256-bit epilogue stores (default) vs two 16-B stores (st128 build): tests + bench lines with training
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py -m gpu -q -x -p no:cacheprovider > gpurun_out/st256_tests.log 2>&1
echo "st256 tests rc=$? $(tail -1 gpurun_out/st256_tests.log)"
for v in default st128 default st128; do
  if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
  NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 > gpurun_out/st_$v.json 2>&1
  python - <<PY
import json
j = json.loads(open("gpurun_out/st_$v.json").read().strip().splitlines()[-1])
s = j["stages"]
print("$v: step %.4f ms gemm1 %.1f gemm2 %.1f comb %.1f | train %.3f %s" % (
    j["ms_per_step"], s["gemm1_ms"] * 1e3, s["gemm2_ms"] * 1e3, s["combine_ms"] * 1e3,
    j["train"]["ms_per_step"], {k: round(v * 1e3) for k, v in j["train"]["bwd_stages_ms"].items()}))
PY
done
