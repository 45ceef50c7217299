cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
true
timeout 600 ncu --replay-mode range --metrics nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,gpu__time_duration.sum --csv --log-file gpurun_out/nvl_ce_ncu.csv python tools/nvlink_ce_probe.py > gpurun_out/nvl_ce_ncu.log 2>&1
echo "rc=$?" >> gpurun_out/nvl_ce_ncu.log
