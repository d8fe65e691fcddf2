# Final 4-GPU evidence with the round-2 kernels and the piece queue default (piece_queue 2).
set -x
export RS_BARRIER_TIMEOUT_S=30
timeout 2400 python -m pytest tests -m gpu -v -rs > gpurun_out/r02d_pytest_gpu_4_final.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02d_pytest_gpu_4_final.log
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29711 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02d_bench_n4_final.log 2>&1; echo "n4 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29712 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02d_bench_n2_final.log 2>&1; echo "n2 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29713 bench.py --gpus 4 --workload kN --steps 3 --warmup 3 --no-e2e --no-rescore-all > gpurun_out/r02d_bench_k4_final.log 2>&1; echo "k4 rc=$?"
for K in 4 2; do
timeout 900 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2972$K tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter,Reduce --reduce-modes=-1 --min-bytes 1048576 --max-bytes 1073741824 --step 4 --iters 20 --out gpurun_out/r02d_collectives_final_k$K.json > gpurun_out/r02d_collectives_final_k$K.log 2>&1; echo "coll K=$K rc=$?"
[ $K = 4 ] && timeout 1800 torchrun --nnodes=1 --nproc-per-node $K --master-addr 127.0.0.1 --master-port 2973$K bench_sweep.py --graph --step 4 --out gpurun_out/r02d_sweep_final_k$K.json > gpurun_out/r02d_sweep_final_k$K.log 2>&1; echo "sweep K=$K rc=$?"
done
for f in r02d_bench_n4_final r02d_bench_n2_final r02d_bench_k4_final; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d.get('speedup_vs_nccl'))" gpurun_out/$f.log; done
for K in 4; do python -c "
import json,sys
d=json.load(open(sys.argv[1]))
for r in d['rows']: print(f\"{r['bytes']:>11} best {r['best_us']:9.1f} nccl {r['nccl_us']:9.1f} x{r['speedup_vs_nccl']:.2f} busbw {r['best_busbw']:6.1f}\")" gpurun_out/r02d_sweep_final_k$K.json; done
