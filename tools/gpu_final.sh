# round-end evidence on one B200 (usage: bash tools/gpu_final.sh TAG)
cd $GRAFT_REPO_ROOT
TAG=${1:-final}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q --timeout 900 -p no:cacheprovider > gpurun_out/${TAG}_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/${TAG}_tests.log
timeout 600 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${TAG}_smoke.log 2>&1
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/${TAG}_bench.log 2> gpurun_out/${TAG}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 80 --csv --log-file gpurun_out/${TAG}_launches.csv python bench.py --steps 2 --warmup 3 --no-train --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:grouped_gemm_sm100_pair -c 2 -o gpurun_out/${TAG}_gemm python bench.py --steps 1 --warmup 3 --no-train --no-cpu-baseline --no-fp32 > gpurun_out/${TAG}_ncu_gemm.log 2>&1
bash tools/c_sweep.sh > gpurun_out/${TAG}_cfg3_sweep.txt 2>&1
bash tools/cfg5_scale.sh 1 > gpurun_out/${TAG}_cfg5.txt 2>&1
