# 4-GPU lease: full GPU suite (release and checked builds), benches N=4/N=2, NCCL without NVLS, config-4 sweeps.
set -x
export RS_BARRIER_TIMEOUT_S=30
timeout 1800 python -m pytest tests -m gpu -v -rs > gpurun_out/r02_pytest_gpu_4_verbose.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_4_verbose.log
RS_LIB_PATH=$PWD/paper_2110_10548_b200/_lib/libredsynth_b200_checked.so timeout 1800 python -m pytest tests -m gpu -v -rs > gpurun_out/r02_pytest_gpu_4_checked.log 2>&1; echo "checked rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_4_checked.log
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 4 --steps 5 --warmup 3 > gpurun_out/r02_bench_n4.log 2>&1; echo "n4 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 > gpurun_out/r02_bench_n2.log 2>&1; echo "n2 rc=$?"
NCCL_NVLS_ENABLE=0 timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29613 bench.py --gpus 4 --workload kN --steps 3 --warmup 3 --no-e2e --no-rescore-all > gpurun_out/r02_bench_k4_nvls0.log 2>&1; echo "k4 nvls0 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29614 bench.py --gpus 4 --workload kN --steps 3 --warmup 3 --no-e2e --no-rescore-all > gpurun_out/r02_bench_k4.log 2>&1; echo "k4 rc=$?"
timeout 1800 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29615 bench_sweep.py --graph --step 4 --out gpurun_out/r02_sweep_k4.json > gpurun_out/r02_sweep_k4.log 2>&1; echo "sweep4 rc=$?"
timeout 1200 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29616 bench_sweep.py --graph --step 4 --out gpurun_out/r02_sweep_k2.json > gpurun_out/r02_sweep_k2.log 2>&1; echo "sweep2 rc=$?"
NCCL_NVLS_ENABLE=0 timeout 1800 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29617 bench_sweep.py --graph --step 4 --programs first:1 --out gpurun_out/r02_sweep_k4_ncclnvls0.json > gpurun_out/r02_sweep_k4_ncclnvls0.log 2>&1; echo "sweep4 nvls0 rc=$?"
for f in r02_bench_n4 r02_bench_n2 r02_bench_k4_nvls0 r02_bench_k4; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'], d.get('speedup_vs_nccl'), d['simulator_rescoring']['instances'], d['simulator_rescoring']['top_k'], (d.get('e2e') or {}).get('value'))" gpurun_out/$f.log; done
