# A/B: push waves (landing and result traffic overlapped) for AllReduce and Reduce (mode 1) at K=4.
set -x
export RS_BARRIER_TIMEOUT_S=20
for W in 0 1048576 4194304 16777216; do
  timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2953$((W % 7)) tools/collectives_vs_nccl.py --ops AllReduce,Reduce --reduce-modes 0,1,2 --nvls --wave-bytes $W --min-bytes 16777216 --max-bytes 1073741824 --step 4 --out gpurun_out/r02_waves_$W.json > gpurun_out/r02_waves_$W.log 2>&1; echo "W=$W rc=$?"
  grep bytes gpurun_out/r02_waves_$W.log | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print(d['bytes']>>20, {k:(v['ours_us'],v['nccl_us']) for k,v in d.items() if k!='bytes'})"
done
