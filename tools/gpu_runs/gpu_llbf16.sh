export RS_BARRIER_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_emulated_ranks.py tests/test_gpu_parity.py -q -x -k "emulated or one_shot or one_slot or interleaved" > gpurun_out/r02_llbf16_tests.log 2>&1; echo "tests rc=$?"; tail -1 gpurun_out/r02_llbf16_tests.log
for K in 4 2; do
timeout 600 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2981$K tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --reduce-modes=-1 --min-bytes 1024 --max-bytes 262144 --step 4 --iters 20 --out gpurun_out/r02_llbf16_k$K.json > /dev/null 2>&1; echo "K=$K rc=$?"
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(' '.join(f\"{r['bytes']>>10}K:\" + '/'.join(f\"{r[k]['ours_us']:.1f}\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_llbf16_k$K.json
done
