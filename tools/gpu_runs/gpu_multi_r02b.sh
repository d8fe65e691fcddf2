# 4-GPU: remote256 A/B (collectives, K=4 and K=2), full GPU suite, N=4/N=2 benches with the final kernels.
set -x
export RS_BARRIER_TIMEOUT_S=30
for R in 0 1; do
  RS_REMOTE256=$R timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2964$R tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --push-min-bytes -1 --min-bytes 1048576 --max-bytes 268435456 --step 4 --out gpurun_out/r02_r256_$R.json > gpurun_out/r02_r256_$R.log 2>&1; echo "R=$R rc=$?"
  python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(r['bytes']>>20, {k:(v['ours_us'],v['nccl_us']) for k,v in r.items() if k!='bytes'})" gpurun_out/r02_r256_$R.json
done
timeout 2400 python -m pytest tests -m gpu -v -rs > gpurun_out/r02_pytest_gpu_4_final.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_4_final.log
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29651 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02_bench_n4_final.log 2>&1; echo "n4 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29652 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_n2_final.log 2>&1; echo "n2 rc=$?"
for f in r02_bench_n4_final r02_bench_n2_final; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d['simulator_rescoring']['top_k'], d['calibrated_rescoring']['top_k'])" gpurun_out/$f.log; done
