cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in base kb128 intconv kb128_intconv noconv nomma noepi; do
  NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/variants/lib_$v.so timeout 300 python tools/router_variants.py >> gpurun_out/r02f_variants.log 2>&1
done
