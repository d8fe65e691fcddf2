# A/B: dynamic piece queue for push phases x push waves, AllReduce and Reduce at K=4; parity of the push paths.
set -x
export RS_BARRIER_TIMEOUT_S=20
timeout 900 python -m pytest tests/test_gpu_ranks_one_gpu.py tests/test_gpu_parity.py tests/test_gpu_multiprocess.py -m gpu -q -x > gpurun_out/r02_dyn_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02_dyn_parity.log
summ() { python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(r['bytes']>>20, {k:(v['ours_us'],v['nccl_us']) for k,v in r.items() if k!='bytes'})" $1; }
i=0
for cfg in "1 0" "1 4194304" "1 16777216" "0 0"; do
  set -- $cfg; D=$1; W=$2; i=$((i+1))
  RS_DYNAMIC_PIECES=$D timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2955$i tools/collectives_vs_nccl.py --ops AllReduce,Reduce --reduce-modes 0,1,2 --nvls --wave-bytes $W --min-bytes 16777216 --max-bytes 1073741824 --step 4 --out gpurun_out/r02_dyn${D}_w$W.json > gpurun_out/r02_dyn${D}_w$W.log 2>&1; echo "D=$D W=$W rc=$?"
  summ gpurun_out/r02_dyn${D}_w$W.json
done
for W in 0 4; do
timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29561 tools/trace_push.py --op allreduce --mib 64 --wave-mib $W --out gpurun_out/r02_trace_ar64_dyn_w$W.json 2>&1 | grep -v Warn | grep -v "^W1\|\*\*\*"
timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29562 tools/trace_push.py --op reduce --reduce-mode 1 --mib 64 --wave-mib $W --out gpurun_out/r02_trace_red64_dyn_w$W.json 2>&1 | grep -v Warn | grep -v "^W1\|\*\*\*"
done
