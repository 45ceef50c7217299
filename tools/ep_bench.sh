# usage: bash tools/ep_bench.sh N "transports" [extra bench args]
N=$1; TR=$2; shift 2
port=29700
for T in $TR; do
  port=$((port+1))
  timeout 400 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port $port bench.py --gpus $N --steps 10 --warmup 3 --ep-transport $T "$@" > gpurun_out/ep${N}_$T.json 2> gpurun_out/ep${N}_$T.err
  echo "== N=$N $T rc=$?"
  python - <<PY
import json
j = json.loads(open("gpurun_out/ep${N}_$T.json").read().strip().splitlines()[-1])
s = j.get("same_config_1gpu") or {}
eff = j["value"] / ($N * s["value"]) if s else None
print(round(j["ms_per_step"], 3), "eff", eff, j["timeline_ms_rank0"])
PY
done
