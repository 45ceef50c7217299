# backward stage times of the default library and the NIMG_BWD_PROBE variants
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in default probe1 probe2; do
  if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
  NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-fp32 > gpurun_out/bwdprobe_$v.json 2>&1
  python - <<PY
import json
j = json.loads(open("gpurun_out/bwdprobe_$v.json").read().strip().splitlines()[-1])
print("$v", {k: round(v * 1e3, 1) for k, v in j["train"]["bwd_stages_ms"].items()})
PY
done
