# combine occupancy A/B: default (3 resident blocks for the bf16 combine) vs the cbminb1 build; GPU tests that use the combine
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_backward.py tests/test_gpu_dit.py tests/test_gpu_sweep.py -m gpu -q -x -p no:cacheprovider > gpurun_out/cb_tests.log 2>&1
echo "tests rc=$? $(tail -1 gpurun_out/cb_tests.log)"
bash tools/gpu_ab_fwd.sh cbminb1 3
