# A/B: AllReduce push waves with 64 KiB reducing pieces at K=4 and K=2 (16 MiB .. 256 MiB).
set -x
export RS_BARRIER_TIMEOUT_S=20
i=0
for K in 4 2; do
for W in 0 1048576 2097152 4194304; do
  i=$((i+1))
  timeout 600 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2960$i tools/collectives_vs_nccl.py --ops AllReduce --wave-bytes $W --push-min-bytes 16777216 --min-bytes 16777216 --max-bytes 268435456 --step 2 --iters 20 --out gpurun_out/r02_arwave${W}_k$K.json > gpurun_out/r02_arwave${W}_k$K.log 2>&1; echo "K=$K W=$W rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(' '.join(f\"{r['bytes']>>20}:{r['AllReduce']['ours_us']}/{r['AllReduce']['nccl_us']}\" for r in d['rows']))" gpurun_out/r02_arwave${W}_k$K.json
done; done
