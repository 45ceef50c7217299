cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
for i in 1 2; do
NIMG_BENCH_DEBUG=1 timeout 900 python bench.py --gpus 4 --steps 20 --warmup 5 > gpurun_out/r02_ep4dbg$i.log 2> gpurun_out/r02_ep4dbg$i.err
done
