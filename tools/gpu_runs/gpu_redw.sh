export RS_BARRIER_TIMEOUT_S=30
i=0
for W in 4194304 1048576 16777216 0; do i=$((i+1))
  timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2969$i tools/collectives_vs_nccl.py --ops Reduce --reduce-modes=-1 --reduce-wave-bytes $W --min-bytes 33554432 --max-bytes 1073741824 --step 2 --iters 10 --out gpurun_out/r02_redw_$W.json > /dev/null 2>&1; echo "W=$W rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') + f\"({list(r.values())[1]['nccl_us']:.0f})\" for r in d['rows']))" gpurun_out/r02_redw_$W.json W=$W
done
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29699 tools/collectives_vs_nccl.py --ops Reduce --reduce-modes=0,1 --min-bytes 33554432 --max-bytes 268435456 --step 2 --iters 10 --out gpurun_out/r02_redw_modes.json > /dev/null 2>&1; echo "modes rc=$?"
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_redw_modes.json
