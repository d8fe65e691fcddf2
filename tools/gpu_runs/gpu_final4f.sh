# Final code on 4 GPUs: full GPU suite, N=4 / N=2 benches (driver-shaped commands).
export RS_BARRIER_TIMEOUT_S=30
timeout 2400 python -m pytest tests -m gpu -v -rs > gpurun_out/r02f_pytest_gpu_4.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02f_pytest_gpu_4.log
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29811 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02f_bench_n4.log 2>&1; echo "n4 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29812 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02f_bench_n2.log 2>&1; echo "n2 rc=$?"
for f in r02f_bench_n4 r02f_bench_n2; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'], (d.get('e2e') or {}).get('value'), d['clocks'])" gpurun_out/$f.log; done
