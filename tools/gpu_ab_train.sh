# alternating A/B of the training step's backward stages: default library vs a variant build (tools/build_variants.py)
# usage: bash tools/gpu_ab_train.sh VARIANT [REPS]
cd $GRAFT_REPO_ROOT
V=$1; REPS=${2:-3}
mkdir -p gpurun_out
for rep in $(seq $REPS); do
  for v in default $V; do
    if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
    NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 > gpurun_out/abt_$v.json 2>&1
    python - <<PY
import json
j = json.loads(open("gpurun_out/abt_$v.json").read().strip().splitlines()[-1])
print("$v rep $rep: step %.4f | train %.3f %s" % (j["ms_per_step"], j["train"]["ms_per_step"],
      {k: round(v * 1e3) for k, v in j["train"]["bwd_stages_ms"].items()}))
PY
  done
done
