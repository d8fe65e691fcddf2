export RS_BARRIER_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_emulated_ranks.py -q -x > gpurun_out/r02_red4_emu.log 2>&1; echo "emu rc=$?"
for i in 1 2; do
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2975$i tools/collectives_vs_nccl.py --ops Reduce --reduce-modes=1,4 --min-bytes 33554432 --max-bytes 1073741824 --step 2 --iters 10 --out gpurun_out/r02_red4_$i.json > /dev/null 2>&1; echo "rc=$?"
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') + f\"({list(r.values())[1]['nccl_us']:.0f})\" for r in d['rows']))" gpurun_out/r02_red4_$i.json
done
