cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_compat.py tests/test_gpu_concurrency.py tests/test_gpu_parity.py -m gpu -q -s --timeout 600 -p no:cacheprovider > gpurun_out/r02b_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02b_tests.log
timeout 900 ncu --set full --import-source on -k regex:router_scores_i8 -c 1 -o gpurun_out/r02b_router python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-train > gpurun_out/r02b_ncu_router.log 2>&1
timeout 600 ncu --set full -k regex:"ec_select|gate_norm|combine_kernel" -c 3 -o gpurun_out/r02b_select python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-train > gpurun_out/r02b_ncu_select.log 2>&1
