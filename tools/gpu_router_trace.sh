# per-CTA %globaltimer traces of the INT8 router (tools/build_variants.py trace variants)
cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
TAG=${1:-trace}
for v in trace trace_nomma trace_noconv; do
  echo "== $v" >> gpurun_out/${TAG}.log
  N=3 NIMG_LIB_PATH=$PWD/paper_2604_12163_b200/libnimg_moe_$v.so timeout 300 python tools/router_variants.py 2>&1 | tail -5 >> gpurun_out/${TAG}.log
done
