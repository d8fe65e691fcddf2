export RS_BARRIER_TIMEOUT_S=30
i=0
for R in 0 1 0 1; do i=$((i+1))
  RS_REMOTE256=$R timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2966$i tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --push-min-bytes -1 --min-bytes 4194304 --max-bytes 268435456 --step 4 --iters 20 --out gpurun_out/r02_r256b_${i}_$R.json > /dev/null 2>&1; echo "R=$R rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_r256b_${i}_$R.json R=$R
done
