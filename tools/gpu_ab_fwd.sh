# alternating forward A/B: default library vs a variant build (tools/build_variants.py); parity tests with the variant
# usage: bash tools/gpu_ab_fwd.sh VARIANT [REPS]
cd $GRAFT_REPO_ROOT
V=$1; REPS=${2:-3}
mkdir -p gpurun_out
NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/libnimg_moe_$V.so timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -p no:cacheprovider > gpurun_out/abf_${V}_tests.log 2>&1
echo "$V parity tests rc=$? $(tail -1 gpurun_out/abf_${V}_tests.log)"
for rep in $(seq $REPS); do
  for v in default $V; do
    if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
    NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-fp32 --no-train > gpurun_out/abf_$v.json 2>&1
    python - <<PY
import json
j = json.loads(open("gpurun_out/abf_$v.json").read().strip().splitlines()[-1])
s = j["stages"]
print("$v rep $rep: step %.4f ms gemm1 %.1f gemm2 %.1f route %.1f comb %.1f" % (j["ms_per_step"], s["gemm1_ms"] * 1e3,
      s["gemm2_ms"] * 1e3, s["route_ms"] * 1e3, s["combine_ms"] * 1e3))
PY
  done
done
