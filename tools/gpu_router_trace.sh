cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for v in trace trace_nomma trace_noconv trace_kb128; do
  echo "== $v" >> gpurun_out/r02h_trace.log
  N=3 NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/variants/lib_$v.so timeout 300 python tools/router_variants.py 2>&1 | tail -5 >> gpurun_out/r02h_trace.log
done
