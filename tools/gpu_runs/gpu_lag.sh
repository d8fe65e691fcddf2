# RS_WAVE_LAG A/B: Reduce push at K=4 (4 MiB waves), 128 MiB - 1 GiB; parity of the lagged order first.
export RS_BARRIER_TIMEOUT_S=20
RS_WAVE_LAG=2 timeout 900 python -m pytest tests/test_gpu_emulated_ranks.py -m gpu -q -x > gpurun_out/r02_lag_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02_lag_parity.log
i=0
for L in 0 1 2 4 0 2; do
  i=$((i+1))
  RS_WAVE_LAG=$L timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2977$i tools/collectives_vs_nccl.py --ops Reduce --reduce-modes=-1 --min-bytes 134217728 --max-bytes 1073741824 --step 2 --iters 20 --out gpurun_out/r02_lag${L}_$i.json > /dev/null 2>&1; echo "L=$L rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[1], [(r['bytes']>>20, [(v['ours_us'], v['nccl_us']) for k,v in r.items() if k!='bytes']) for r in d['rows']])" gpurun_out/r02_lag${L}_$i.json
done
