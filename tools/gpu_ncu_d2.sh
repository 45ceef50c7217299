cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 ncu --set full --import-source on -k regex:"grouped_gemm_bwd_sm100<0" -c 1 -o gpurun_out/r02_d2 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp32 > gpurun_out/r02_d2_ncu.log 2>&1
