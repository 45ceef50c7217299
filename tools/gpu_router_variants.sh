# routing-stage time of INT8-router A/B builds (build them first: python tools/build_variants.py base kb128 ...)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in ${@:-kb128 intconv b128 noconv nomma noepi}; do
  NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/libnimg_moe_$v.so timeout 300 python tools/router_variants.py >> gpurun_out/router_variants.log 2>&1
done
