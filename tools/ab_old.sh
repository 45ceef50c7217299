# Same-box A/B: this tree vs old_tree/ (a git worktree of an older commit).
one() {  # $1 = dir, $2 = label, $3 = env
  (cd $1 && env $3 python bench.py --steps 20 --warmup 5 --no-cpu-baseline 2>/dev/null) | python -c "
import json,sys; j=json.loads(sys.stdin.read().strip().splitlines()[-1]); s=j['stages']
print('$2 ms %.4f route %.4f g1 %.4f g2 %.4f comb %.4f gather %.4f block %.4f' % (j['ms_per_step'], s['route_ms'], s['gemm1_ms'], s['gemm2_ms'], s['combine_ms'], s['gather_ms'], j['block']['ms_per_step']), s.get('router_scores_ms'))"
}
for i in 1 2; do
  one old_tree old NIMG_X=1
  one . new_pdl NIMG_PDL=1
  one . new_nopdl NIMG_PDL=0
done
