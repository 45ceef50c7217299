# A/B of programmatic dependent launch on the cfg2 bench (1 GPU).
for i in 1 2; do
  for pdl in 1 0; do
    NIMG_PDL=$pdl python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=j['stages']
print('pdl=$pdl ms %.4f route %.4f scores %.4f sel %.4f gather %.4f g1 %.4f g2 %.4f comb %.4f block %.4f e2e %.4g' % (j['ms_per_step'], s['route_ms'], s['router_scores_ms'], s['select_gates_ms'], s['gather_ms'], s['gemm1_ms'], s['gemm2_ms'], s['combine_ms'], j['block']['ms_per_step'], j['e2e']['value']))"
  done
done
