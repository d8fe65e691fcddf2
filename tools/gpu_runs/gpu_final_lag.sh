# Final code (wave_lag 2): 4-GPU cross-rank parity suites and the K=4/K=2 per-collective table.
export RS_BARRIER_TIMEOUT_S=30
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multiprocess.py tests/test_gpu_ranks_processes.py tests/test_gpu_nvls.py -m gpu -q -rs > gpurun_out/r02g_pytest_gpu_4_cross.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02g_pytest_gpu_4_cross.log
for K in 4 2; do
timeout 900 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2982$K tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --reduce-modes=-1 --min-bytes 1048576 --max-bytes 1073741824 --step 4 --iters 20 --out gpurun_out/r02g_collectives_k$K.json > gpurun_out/r02g_collectives_k$K.log 2>&1; echo "coll K=$K rc=$?"
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(r['bytes']>>20, {k:(v['ours_us'],v['nccl_us']) for k,v in r.items() if k!='bytes'})" gpurun_out/r02g_collectives_k$K.json
done
