# cfg5 stack (Nucleus-Image, 1024px stage) at N = 1, 2, 4 GPUs, B=4 per GPU.
mkdir -p gpurun_out
for N in "$@"; do
  if [ "$N" = 1 ]; then
    timeout 900 python bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/cfg5_n1.json 2> gpurun_out/cfg5_n1.err
  else
    timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 \
      --master-port $((29600 + N)) bench.py --config cfg5 --steps 5 --warmup 3 > gpurun_out/cfg5_n$N.json 2> gpurun_out/cfg5_n$N.err
  fi
  echo "== N=$N rc=$?"
  python -c "
import json; j=json.loads(open('gpurun_out/cfg5_n$N.json').read().strip().splitlines()[-1])
print('N=$N ms %.2f tok/s %.4g' % (j['ms_per_step'], j['value']), j['phase_ms_rank0'])"
done
