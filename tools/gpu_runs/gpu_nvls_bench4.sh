# De-risk the N=8 bench flow: NVLS forced for the 4-GPU groups (multicast setup + self-check through the NCCL
# process group exchange, in bench.py's own flow), config 2 at N=4 and config-4 K=4.
export RS_BARRIER_TIMEOUT_S=30
RS_NVLS_MIN_BYTES=0 timeout 1500 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29801 bench.py --gpus 4 --steps 3 --warmup 3 > gpurun_out/r02_bench_n4_nvlsforced.log 2>&1; echo "n4 nvls rc=$?"
RS_NVLS_MIN_BYTES=0 timeout 1500 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29802 bench.py --gpus 4 --workload kN --steps 3 --warmup 3 --no-e2e > gpurun_out/r02_bench_k4_nvlsforced.log 2>&1; echo "k4 nvls rc=$?"
for f in r02_bench_n4_nvlsforced r02_bench_k4_nvlsforced; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('nvls'), d.get('speedup_vs_nccl'), (d.get('e2e') or {}).get('value'))" gpurun_out/$f.log; tail -3 gpurun_out/$f.log | cut -c1-300; done
