cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
N=3 NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/variants/lib_trace.so timeout 300 python tools/router_variants.py 2>&1 | tail -3 >> gpurun_out/r02k.log
