# one iteration: routing + backward GPU tests, a bench line, and the cfg2 launch list
# (usage: bash tools/gpu_iter.sh TAG)
cd $GRAFT_REPO_ROOT
TAG=${1:-iter}
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_router_i8.py tests/test_gpu_parity.py tests/test_gpu_backward.py -m gpu -q -x \
  --timeout 600 -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_bench.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/${TAG}_launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_ncu.log 2>&1
