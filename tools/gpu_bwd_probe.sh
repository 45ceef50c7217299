# backward stage times of the default library and variant builds (tools/build_variants.py)
# usage: bash tools/gpu_bwd_probe.sh [variant ...]   (default: probe1 probe2)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
VARS=${@:-probe1 probe2}
for v in default $VARS; do
  if [ $v = default ]; then lib=paper_2604_12163_b200/libnimg_moe.so; else lib=paper_2604_12163_b200/libnimg_moe_$v.so; fi
  case $v in probe*) ;; *)
    NIMG_LIB_PATH=$PWD/$lib timeout 600 python -m pytest tests/test_gpu_backward.py -m gpu -q -x -p no:cacheprovider \
      > gpurun_out/bwdprobe_${v}_tests.log 2>&1; echo "$v tests rc=$? $(tail -1 gpurun_out/bwdprobe_${v}_tests.log)";;
  esac
  NIMG_LIB_PATH=$PWD/$lib timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-fp32 > gpurun_out/bwdprobe_$v.json 2>&1
  python - <<PY
import json
j = json.loads(open("gpurun_out/bwdprobe_$v.json").read().strip().splitlines()[-1])
print("$v", {k: round(v * 1e3, 1) for k, v in j["train"]["bwd_stages_ms"].items()})
PY
done
