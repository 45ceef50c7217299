cd $GRAFT_REPO_ROOT
TAG=${1:-q2}
mkdir -p gpurun_out
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_ep.py tests/test_gpu_graph.py tests/test_gpu_concurrency.py tests/test_gpu_dit.py -m gpu -q -x --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python bench.py --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_bench.log 2>&1
NIMG_TOK_ORDER=1 timeout 600 python bench.py --steps 20 --warmup 5 --no-train --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_bench_notok.log 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_ncu.log 2>&1
