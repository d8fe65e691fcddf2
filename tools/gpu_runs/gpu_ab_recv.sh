# A/B: push reducing piece 64 KiB (default) vs 256 KiB (= flag chunk), K=4 and K=2; quick parity of the push path.
set -x
export RS_BARRIER_TIMEOUT_S=20
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py -m gpu -q -x -k "push or two_gpus or one_slot or interleaved or three or ipc" > gpurun_out/r02_recv_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02_recv_parity.log
i=0
for K in 4 2; do
for RP in 65536 262144; do
  i=$((i+1))
  RS_RECV_PIECE=$RP timeout 600 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2959$i tools/collectives_vs_nccl.py --ops AllReduce,Reduce --min-bytes 16777216 --max-bytes 1073741824 --step 2 --out gpurun_out/r02_recv${RP}_k$K.json > gpurun_out/r02_recv${RP}_k$K.log 2>&1; echo "K=$K RP=$RP rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(r['bytes']>>20, {k:(v['ours_us'],v['nccl_us'],v['task_modes']) for k,v in r.items() if k!='bytes'})" gpurun_out/r02_recv${RP}_k$K.json
done; done
