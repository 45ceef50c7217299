# capacity-factor sweep at 1024px (S=4096, B=16), 1 GPU.
# usage: bash tools/c_sweep.sh   (writes gpurun_out/cfg3_C*.json)
mkdir -p gpurun_out
for C in 8 4 2; do
  timeout 600 python bench.py --config cfg3 --capacity $C --steps 10 --warmup 3 --no-cpu-baseline --no-train --no-fp32 \
    > gpurun_out/cfg3_C$C.json 2> gpurun_out/cfg3_C$C.err
  echo "== C=$C rc=$?"
  python - <<PY
import json
j = json.loads(open("gpurun_out/cfg3_C$C.json").read().strip().splitlines()[-1])
s = j["stages"]
print("C=$C ms %.3f tok/s %.4g gemm TF %.0f (%.2f of peak) router %.3f ms (%.1f f64-equiv TF/s) sel %.3f gather %.3f g1 %.3f g2 %.3f comb %.3f" % (
    j["ms_per_step"], j["value"], j["expert_gemm_tflops"], j["expert_gemm_frac_of_peak"],
    s["router_scores_ms"], s["router_f64_equiv_tflops"], s["select_gates_ms"], s["gather_ms"],
    s["gemm1_ms"], s["gemm2_ms"], s["combine_ms"]))
PY
done
