cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:"router_scores_i8|ec_select_warp|gate_tile" -c 3 -o gpurun_out/r02d_route python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-train > gpurun_out/r02d_ncu.log 2>&1
