# full ncu captures of the routing kernels and the combine at cfg2 (usage: bash tools/gpu_ncu_route.sh TAG)
cd $GRAFT_REPO_ROOT
TAG=${1:-route}
mkdir -p gpurun_out
timeout 900 ncu --set full --clock-control none --import-source on -k regex:"router_scores_i8|ec_select_blk|gate_tile|combine_kernel" -c 4 \
  -o gpurun_out/${TAG} python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-train --no-fp32 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
