# AllReduce push waves with wave_lag 2 (waves alone were slower in round 2): K=4, 64 MiB - 1 GiB; parity first.
export RS_BARRIER_TIMEOUT_S=20
RS_PUSH_WAVE_BYTES=4194304 timeout 600 python -m pytest tests/test_gpu_emulated_ranks.py -m gpu -q -x -k "full_size or every_variant" > gpurun_out/r02_arwl_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02_arwl_parity.log
i=0
for W in 0 4194304 16777216 0; do
  i=$((i+1))
  RS_PUSH_WAVE_BYTES=$W timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2983$i tools/collectives_vs_nccl.py --ops AllReduce --min-bytes 67108864 --max-bytes 1073741824 --step 4 --iters 20 --out gpurun_out/r02_arwl_$W_$i.json > /dev/null 2>&1; echo "W=$W rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], [(r['bytes']>>20, [v['ours_us'] for k,v in r.items() if k!='bytes']) for r in d['rows']])" gpurun_out/r02_arwl_$W_$i.json $W
done
