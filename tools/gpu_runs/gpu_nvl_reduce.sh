# NVLink + DRAM bytes of the K=4 256 MiB Reduce launches (push = default at this size, and pull), and of the
# K=4 push AllReduce for comparison, one GPU's launch replayed alone (profiling build, RS_SOLO_PROFILE=1).
ncu --query-metrics 2>/dev/null | grep -i "^nvl" > gpurun_out/r02_nvl_metric_names.txt
M=gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,nvltx__bytes_data_user.sum,nvlrx__bytes_data_user.sum,dram__bytes_read.sum,dram__bytes_write.sum
for spec in "Reduce 1 1" "Reduce 0 0" "AllReduce 1 -1"; do
  set -- $spec
  RS_SOLO_PROFILE=1 timeout 600 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/r02_nvl_$1_push$2.csv \
    python tools/profile_p2p.py --gpus 4 --op $1 --push $2 --reduce-mode $3 > gpurun_out/r02_nvl_$1_push$2.log 2>&1
  echo "$spec rc=$?"; tail -2 gpurun_out/r02_nvl_$1_push$2.log
done
