# A/B of library variants on the training leg of the cfg2 bench (1 GPU).
#   usage: bash tools/ab_train.sh libA.so libB.so [...]   (paths relative to repo root)
for i in 1 2; do
  for lib in "$@"; do
    NIMG_LIB_PATH=$PWD/$lib python bench.py --steps 10 --warmup 3 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); t=j['train']; s=t['bwd_stages_ms']
print('$lib', 'fwd %.3f bwd %.3f' % (j['ms_per_step'], t['bwd_ms']), ' '.join('%s %.3f' % (k[:8], v) for k, v in s.items()))"
  done
done
