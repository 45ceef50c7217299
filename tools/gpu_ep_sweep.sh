# EP4 schedule sweep: NIMG_EP_RET_SPLIT x NIMG_EP_OWN_A, then the EP tests (usage: bash tools/gpu_ep_sweep.sh TAG)
cd $GRAFT_REPO_ROOT
TAG=${1:-eps}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_ep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
for cfg in "1 -1" "2 -1" "2 4" "3 -1" "2 6"; do
  set -- $cfg
  NIMG_EP_RET_SPLIT=$1 NIMG_EP_OWN_A=$2 timeout 600 python bench.py --gpus 4 --steps 20 --warmup 5 \
    > gpurun_out/${TAG}_r$1_a$2.json 2> gpurun_out/${TAG}_r$1_a$2.err
  python - <<PY
import json
try:
    j = json.loads(open("gpurun_out/${TAG}_r$1_a$2.json").read().strip().splitlines()[-1])
    c = j.get("cfg4_strong", {})
    print("split $1 own_a $2: weak %.4f ms, cfg4 %.4f ms" % (j["ms_per_step"], c.get("ms_per_step", float("nan"))))
except Exception as e:
    print("split $1 own_a $2: failed", e)
PY
done
