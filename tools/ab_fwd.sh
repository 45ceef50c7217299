# A/B of library variants on the forward stages of the cfg2 bench (1 GPU).
#   usage: bash tools/ab_fwd.sh libA.so libB.so [...]
for i in 1 2; do
  for lib in "$@"; do
    NIMG_LIB_PATH=$PWD/$lib python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-train 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=j['stages']
print('$lib', 'ms %.4f' % j['ms_per_step'], ' '.join('%s %.4f' % (k, v) for k, v in s.items() if k.endswith('_ms')))"
  done
done
