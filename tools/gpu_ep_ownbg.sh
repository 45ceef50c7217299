# EP: own-chunk background gather (NIMG_EP_OWN_BG=1) vs the gather kernel for every chunk
# usage: bash tools/gpu_ep_ownbg.sh N TAG
cd $GRAFT_REPO_ROOT
N=${1:-4}; TAG=${2:-ownbg}
mkdir -p gpurun_out
NIMG_EP_OWN_BG=1 timeout 1200 python -m pytest tests/test_gpu_ep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "own-bg EP tests rc=$? $(tail -1 gpurun_out/${TAG}_tests.log)"
for rep in 1 2; do
  for v in 0 1; do
    NIMG_EP_OWN_BG=$v timeout 900 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_own$v.json 2> gpurun_out/${TAG}_own$v.err
    python - <<PY
import json
j = json.loads(open("gpurun_out/${TAG}_own$v.json").read().strip().splitlines()[-1])
c = j.get("cfg4_strong", {})
print("own_bg=$v rep $rep: weak %.4f ms, cfg4 %.4f ms (1-GPU %.4f)" % (j["ms_per_step"], c.get("ms_per_step", float("nan")),
      c.get("same_config_1gpu", {}).get("ms_per_step", float("nan"))))
PY
  done
done
