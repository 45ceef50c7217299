cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in base trace; do
  N=3 NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/variants/lib_$v.so timeout 300 python tools/router_variants.py 2>&1 | tail -3 >> gpurun_out/r02m.log
done
timeout 900 python -m pytest tests/test_gpu_router_i8.py tests/test_gpu_parity.py -m gpu -q -x --timeout 600 -p no:cacheprovider -k "route or router or full_width or golden or tie or nan" >> gpurun_out/r02m.log 2>&1
