export RS_BARRIER_TIMEOUT_S=30
i=0
for G in 1 0 1 0; do i=$((i+1))
RS_LANDING_FULL_GRID=$G timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2983$i tools/collectives_vs_nccl.py --ops Reduce --reduce-modes=-1 --min-bytes 134217728 --max-bytes 1073741824 --step 2 --iters 10 --out gpurun_out/r02_rootgrid_${i}_$G.json > /dev/null 2>&1
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_rootgrid_${i}_$G.json G=$G
done
