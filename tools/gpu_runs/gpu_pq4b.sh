# Same-box ABAB: piece_queue 1 vs 2 (pull/NVLS phases queued above 2 pieces per CTA), K=4 collectives and N=4/N=2 benches.
export RS_BARRIER_TIMEOUT_S=30
i=0
for Q in 1 2 1 2; do
  i=$((i+1))
  RS_PIECE_QUEUE=$Q timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2974$i tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --reduce-modes=-1 --min-bytes 4194304 --max-bytes 268435456 --step 4 --iters 20 --out gpurun_out/r02_pqb${Q}_$i.json > /dev/null 2>&1; echo "coll Q=$Q rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[1], [(r['bytes']>>20, [v['ours_us'] for k,v in r.items() if k!='bytes']) for r in d['rows']])" gpurun_out/r02_pqb${Q}_$i.json
done
for Q in 1 2 1 2; do
  i=$((i+1))
  for N in 4 2; do
  RS_PIECE_QUEUE=$Q timeout 900 torchrun --nnodes=1 --nproc-per-node $N --master-addr 127.0.0.1 --master-port 297$N$i bench.py --gpus $N --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pqb${Q}_n${N}_$i.log 2>&1
  python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'])" gpurun_out/r02_pqb${Q}_n${N}_$i.log
  done
done
