cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for bgv in 1 0; do
  NIMG_EP_BG_GATHER=$bgv PYTHONFAULTHANDLER=1 MALLOC_CHECK_=3 timeout 900 python bench.py --gpus 2 --steps 20 --warmup 5 > gpurun_out/r02_ep2d_bg$bgv.log 2> gpurun_out/r02_ep2d_bg$bgv.err
  echo "rc=$?" >> gpurun_out/r02_ep2d_bg$bgv.err
done
