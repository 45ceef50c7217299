# usage: bash tools/ep_bench.sh N [extra bench args]
N=$1; shift
port=$((29700 + N))
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 10 --warmup 3 "$@" > gpurun_out/ep${N}.json 2> gpurun_out/ep${N}.err
echo "== N=$N rc=$?"
python - <<PY
import json
j = json.loads(open("gpurun_out/ep${N}.json").read().strip().splitlines()[-1])
print("weak: ms %.3f value %.4g host %s" % (j["ms_per_step"], j["value"], j.get("host_issue_ms_rank0")), j["timeline_ms_rank0"])
s = j.get("cfg4_strong")
if s:
    print("cfg4 strong: ms %.3f eff %s" % (s["ms_per_step"], s.get("efficiency")), s["timeline_ms_rank0"])
print("e2e", j["e2e"]["ms_per_step"])
PY
