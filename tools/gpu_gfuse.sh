# gates formed in the combine (default) vs the gate kernel (NIMG_GATES_IN_COMBINE=0): tests + alternating bench
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_router_i8.py tests/test_gpu_compat.py tests/test_gpu_graph.py \
  tests/test_gpu_sweep.py tests/test_gpu_dit.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gfuse_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/gfuse_tests.log)"
for rep in 1 2 3; do
  for v in 1 0; do
    NIMG_GATES_IN_COMBINE=$v timeout 600 python bench.py --steps 30 --warmup 5 --no-cpu-baseline --no-fp32 --no-train > gpurun_out/gf_$v.json 2>&1
    python - <<PY
import json
j = json.loads(open("gpurun_out/gf_$v.json").read().strip().splitlines()[-1])
s = j["stages"]
print("gates_in_combine=$v rep $rep: step %.4f ms route %.1f sel+gates %.1f gemm1 %.1f gemm2 %.1f comb %.1f | block %.4f" % (
    j["ms_per_step"], s["route_ms"] * 1e3, s["select_gates_ms"] * 1e3, s["gemm1_ms"] * 1e3, s["gemm2_ms"] * 1e3,
    s["combine_ms"] * 1e3, j["block"]["ms_per_step"]))
PY
  done
done
