export RS_BARRIER_TIMEOUT_S=30
for i in 1 2 3; do
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2974$i tools/collectives_vs_nccl.py --ops ReduceScatter,AllReduce --min-bytes 4194304 --max-bytes 67108864 --step 2 --iters 20 --out gpurun_out/r02_rs16_$i.json > /dev/null 2>&1
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_rs16_$i.json
done
RS_REMOTE256=0 timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29749 tools/collectives_vs_nccl.py --ops ReduceScatter,AllReduce --min-bytes 4194304 --max-bytes 67108864 --step 2 --iters 20 --out gpurun_out/r02_rs16_r0.json > /dev/null 2>&1
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print('R0', ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_rs16_r0.json
