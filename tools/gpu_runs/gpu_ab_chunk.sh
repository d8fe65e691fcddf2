# A/B: push chunk size x CTAs per SM (dynamic queue on), AllReduce and Reduce (push, 4 MiB waves) at K=4.
set -x
export RS_BARRIER_TIMEOUT_S=20
i=0
for cfg in "262144 0" "131072 0" "65536 0" "262144 296" "131072 296"; do
  set -- $cfg; C=$1; M=$2; i=$((i+1))
  RS_FLAG_CHUNK=$C RS_MAX_CTAS=$M timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2957$i tools/collectives_vs_nccl.py --ops AllReduce,Reduce --reduce-modes 1 --wave-bytes 4194304 --min-bytes 16777216 --max-bytes 1073741824 --step 4 --out gpurun_out/r02_chunk${C}_ctas$M.json > gpurun_out/r02_chunk${C}_ctas$M.log 2>&1; echo "C=$C M=$M rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(r['bytes']>>20, {k:(v['ours_us'],v['nccl_us']) for k,v in r.items() if k!='bytes'})" gpurun_out/r02_chunk${C}_ctas$M.json
done
timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29581 tools/trace_push.py --op reduce --reduce-mode 1 --mib 1024 --wave-mib 4 --out gpurun_out/r02_trace_red1g_dyn_w4.json 2>&1 | grep -v Warn | grep -v "^W1\|\*\*\*"
timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29582 tools/trace_push.py --op allreduce --mib 1024 --out gpurun_out/r02_trace_ar1g_dyn.json 2>&1 | grep -v Warn | grep -v "^W1\|\*\*\*"
