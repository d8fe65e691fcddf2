# push_prefetch A/B (push phases reserve their next piece ahead), 4 GPUs: parity first, then ABAB.
export RS_BARRIER_TIMEOUT_S=20
RS_PUSH_PREFETCH=1 timeout 1200 python -m pytest tests/test_gpu_emulated_ranks.py tests/test_gpu_parity.py tests/test_gpu_multiprocess.py tests/test_gpu_ranks_processes.py -m gpu -q -x > gpurun_out/r02_pushpf_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02_pushpf_parity.log
i=0
for F in 0 1 0 1; do
  i=$((i+1))
  RS_PUSH_PREFETCH=$F timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2975$i tools/collectives_vs_nccl.py --ops AllReduce,Reduce --reduce-modes=-1 --min-bytes 16777216 --max-bytes 1073741824 --step 4 --iters 20 --out gpurun_out/r02_pushpf${F}_$i.json > /dev/null 2>&1; echo "coll F=$F rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[1], [(r['bytes']>>20, [v['ours_us'] for k,v in r.items() if k!='bytes']) for r in d['rows']])" gpurun_out/r02_pushpf${F}_$i.json
done
for F in 0 1 0 1; do
  i=$((i+1))
  RS_PUSH_PREFETCH=$F timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2976$i bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pushpf${F}_n4_$i.log 2>&1
  python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'])" gpurun_out/r02_pushpf${F}_n4_$i.log
done
