# flag chunk 128 KiB vs 256 KiB (push path), K=4 and K=2.
export RS_BARRIER_TIMEOUT_S=30
i=0
for K in 4 2; do
for FC in 131072 262144 131072 262144; do i=$((i+1))
  RS_FLAG_CHUNK=$FC timeout 600 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2976$i tools/collectives_vs_nccl.py --ops AllReduce,Reduce --reduce-modes=-1 --min-bytes 33554432 --max-bytes 1073741824 --step 2 --iters 10 --out gpurun_out/r02_fc_${K}_${i}_$FC.json > /dev/null 2>&1; echo "K=$K FC=$FC rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_fc_${K}_${i}_$FC.json "K=$K FC=$FC"
done; done
