cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/r02a_tests.log 2>&1
echo "tests rc=$?" >> gpurun_out/r02a_tests.log
for tool in racecheck synccheck memcheck; do
  timeout 900 /usr/local/cuda/bin/compute-sanitizer --tool $tool --print-limit 50 python tools/sanitize_case.py > gpurun_out/r02a_sanitize_$tool.log 2>&1
  echo "rc=$?" >> gpurun_out/r02a_sanitize_$tool.log
done
timeout 600 python bench.py --steps 20 --warmup 5 > gpurun_out/r02a_bench.log 2>&1
