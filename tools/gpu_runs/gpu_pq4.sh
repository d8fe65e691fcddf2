# 4 GPUs: piece_queue A/B (0 static / 1 own-HBM phases / 2 also pull+NVLS) on the N=4 and N=2 benches
# and per collective at K=4; full GPU suite with the new default.
export RS_BARRIER_TIMEOUT_S=30
summ() { python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" $1; }
for Q in 0 1 2; do
  RS_PIECE_QUEUE=$Q timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2971$Q bench.py --gpus 4 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pq${Q}_n4.log 2>&1; echo "n4 Q=$Q rc=$?"; summ gpurun_out/r02_pq${Q}_n4.log
  RS_PIECE_QUEUE=$Q timeout 900 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 2972$Q bench.py --gpus 2 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pq${Q}_n2.log 2>&1; echo "n2 Q=$Q rc=$?"; summ gpurun_out/r02_pq${Q}_n2.log
done
for Q in 1 2; do
  RS_PIECE_QUEUE=$Q timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2973$Q tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,AllGather,Reduce,Broadcast --min-bytes 1048576 --max-bytes 268435456 --step 4 --out gpurun_out/r02_pq${Q}_coll4.json > gpurun_out/r02_pq${Q}_coll4.log 2>&1; echo "coll Q=$Q rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(r['bytes']>>20, {k:(v['ours_us'],v['nccl_us']) for k,v in r.items() if k!='bytes'})" gpurun_out/r02_pq${Q}_coll4.json
done
timeout 2400 python -m pytest tests -m gpu -q -rs > gpurun_out/r02_pytest_gpu_4_pq.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_gpu_4_pq.log
