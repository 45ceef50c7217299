cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 ncu --set full --import-source on -k regex:"grouped_gemm_bwd" -c 4 -o gpurun_out/r02_bwd python bench.py --steps 1 --warmup 3 --no-cpu-baseline > gpurun_out/r02_bwd_ncu.log 2>&1
