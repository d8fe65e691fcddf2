# One-shot (LL) budget sweep at K=4 and K=2: AllReduce / ReduceScatter / Reduce, 4 KiB .. 2 MiB.
set -x
export RS_BARRIER_TIMEOUT_S=20
i=0
for K in 4 2; do
for LL in 0 16384 32768 65536 262144; do
  i=$((i+1))
  timeout 600 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2962$i tools/collectives_vs_nccl.py --ll-max-bytes $LL --min-bytes 4096 --max-bytes 2097152 --step 2 --iters 20 --out gpurun_out/r02_llb${LL}_k$K.json > gpurun_out/r02_llb${LL}_k$K.log 2>&1; echo "K=$K LL=$LL rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(' '.join(f\"{r['bytes']>>10}K:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in ('AllReduce','ReduceScatter','Reduce')) for r in d['rows']))" gpurun_out/r02_llb${LL}_k$K.json
done; done
