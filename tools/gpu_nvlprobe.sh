cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 300 python tools/nvlink_probe.py > gpurun_out/nvlink_probe.log 2>&1
nvidia-smi nvlink -h > gpurun_out/nvlink_help.txt 2>&1
