# expert-parallel tests + bench on N GPUs of one box (usage: bash tools/gpu_ep.sh N TAG)
cd $GRAFT_REPO_ROOT
N=${1:-2}; TAG=${2:-ep$N}
mkdir -p gpurun_out
nvidia-smi topo -m > gpurun_out/${TAG}_topo.txt 2>&1
timeout 1200 python -m pytest tests/test_gpu_ep.py -m gpu -q -s --timeout 1000 -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 1200 python bench.py --gpus $N --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
echo "bench rc=$?" >> gpurun_out/${TAG}_bench.err
