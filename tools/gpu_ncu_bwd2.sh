# full ncu captures of the five backward grouped GEMM launches of one training step
# (usage: bash tools/gpu_ncu_bwd2.sh TAG)
cd $GRAFT_REPO_ROOT
TAG=${1:-bwd2}
mkdir -p gpurun_out
timeout 600 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_bench.log 2>&1
timeout 1500 ncu --set full --import-source on --clock-control none -k regex:"grouped_gemm_bwd" -c 5 \
  -o gpurun_out/${TAG} python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_ncu.log 2>&1
echo "ncu rc=$?" >> gpurun_out/${TAG}_ncu.log
