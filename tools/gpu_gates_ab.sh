# gate kernels A/B: thread per token (default) vs warp per token (NIMG_GATES=tile)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_router_i8.py tests/test_gpu_ep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/gates_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/gates_tests.log)"
for v in tok tile tok tile; do
  if [ $v = tile ]; then export NIMG_GATES=tile; else unset NIMG_GATES; fi
  timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 --no-train > gpurun_out/gates_$v.json 2>&1
  python - <<PY
import json
j = json.loads(open("gpurun_out/gates_$v.json").read().strip().splitlines()[-1])
s = j["stages"]
print("$v: step %.4f ms route %.1f router %.1f select+gates %.1f" % (
    j["ms_per_step"], s["route_ms"] * 1e3, s["router_scores_ms"] * 1e3, s["select_gates_ms"] * 1e3))
PY
done
unset NIMG_GATES
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"gate_|select" -c 12 --csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fp32 --no-train > gpurun_out/gates_ncu.csv 2>/dev/null
grep -E "gate_|select" gpurun_out/gates_ncu.csv | awk -F'","' '{print $5, $NF}' | head -12
