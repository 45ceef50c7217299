run() { # $1 tag, rest env
  tag=$1; shift
  env "$@" timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port $((29600 + RANDOM % 300)) bench.py --gpus 4 --steps 10 --warmup 3 --no-same-config-1gpu > gpurun_out/exp_$tag.json 2> gpurun_out/exp_$tag.err
  echo "== $tag rc=$?"
  python -c "
import json; j=json.loads(open('gpurun_out/exp_$tag.json').read().strip().splitlines()[-1]); print(round(j['ms_per_step'],3), j['timeline_ms_rank0'])"
}
run base
run ceMemcpy NCCL_P2P_USE_CUDA_MEMCPY=1
run sms132 NIMG_GEMM_MAX_SMS=132
run sms132ch8 NIMG_GEMM_MAX_SMS=132 NCCL_MAX_NCHANNELS=8
