# A/B of library variants (tools/build_variants.py): parity + backward tests and a bench line each
# usage: bash tools/gpu_variants.sh TAG variant ...
cd $GRAFT_REPO_ROOT
TAG=$1; shift
mkdir -p gpurun_out
for v in default "$@"; do
  if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
  if [ $v != default ]; then
    NIMG_LIB_PATH=$PWD/$lib timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py tests/test_gpu_compat.py \
      -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_${v}_tests.log 2>&1
    echo "$v tests rc=$? $(tail -1 gpurun_out/${TAG}_${v}_tests.log)"
  fi
  for rep in 1 2; do
    NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_${v}_$rep.json 2>&1
    python - <<PY
import json
j = json.loads(open("gpurun_out/${TAG}_${v}_$rep.json").read().strip().splitlines()[-1])
s = j["stages"]
print("$v rep $rep: step %.4f ms gemm1 %.1f gemm2 %.1f route %.1f | train %.3f ms %s" % (
    j["ms_per_step"], s["gemm1_ms"] * 1e3, s["gemm2_ms"] * 1e3, s["route_ms"] * 1e3,
    j["train"]["ms_per_step"], {k: round(v * 1e3) for k, v in j["train"]["bwd_stages_ms"].items()}))
PY
  done
done
