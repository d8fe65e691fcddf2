export RS_BARRIER_TIMEOUT_S=30
timeout 1200 python -m pytest tests/test_gpu_emulated_ranks.py tests/test_gpu_parity.py tests/test_gpu_multiprocess.py tests/test_gpu_ranks_processes.py -m gpu -q -x > gpurun_out/r02_r256_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02_r256_parity.log
i=0
for R in 0 1 0 1; do i=$((i+1))
  RS_REMOTE256=$R timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2967$i tools/collectives_vs_nccl.py --ops AllReduce,Reduce --reduce-modes -1 --min-bytes 33554432 --max-bytes 1073741824 --step 2 --iters 10 --out gpurun_out/r02_r256c_${i}_$R.json > /dev/null 2>&1; echo "R=$R rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_r256c_${i}_$R.json R=$R
done
