cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_backward.py tests/test_gpu_guards.py -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r02_bwd_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_bwd_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-cpu-baseline --no-fp32 > gpurun_out/r02_bwd_bench.log 2>&1
