# A/B: cross-GPU pull sums with every source's loads in flight (RS_WIDE_LOADS=1) vs serialized per source.
set -x
export RS_BARRIER_TIMEOUT_S=20
timeout 600 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "two_gpus or one_slot or config3_programs_across or three_gpus or interleaved" > gpurun_out/r02_wide_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02_wide_parity.log
for W in 1 0; do
  RS_WIDE_LOADS=$W timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2952$W tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --reduce-modes 0,2 --nvls --push-min-bytes -1 --min-bytes 1048576 --max-bytes 1073741824 --step 4 --out gpurun_out/r02_wide$W.json > gpurun_out/r02_wide$W.log 2>&1; echo "wide=$W rc=$?"
  grep bytes gpurun_out/r02_wide$W.log
done
