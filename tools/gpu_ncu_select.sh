cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:"ec_select|gate_tile|combine_kernel" -c 3 -o gpurun_out/r02n_select python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-train > gpurun_out/r02n_ncu.log 2>&1
