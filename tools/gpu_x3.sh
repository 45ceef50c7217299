cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "fp32" > gpurun_out/r02_x3_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02_x3_tests.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-train > gpurun_out/r02_x3_bench.log 2>&1
