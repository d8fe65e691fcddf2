# Per-program device times (configs 1-3) at N=4 and N=2 for the cost-model fit.
export RS_BARRIER_TIMEOUT_S=30
timeout 1500 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29781 bench.py --gpus 4 --steps 3 --warmup 3 --no-e2e --programs-out gpurun_out/r02_programs_n4.json > gpurun_out/r02_bench_n4_progs.log 2>&1; echo "n4 rc=$?"
timeout 1500 torchrun --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29782 bench.py --gpus 2 --steps 3 --warmup 3 --no-e2e --programs-out gpurun_out/r02_programs_n2.json > gpurun_out/r02_bench_n2_progs.log 2>&1; echo "n2 rc=$?"
timeout 1500 python bench.py --steps 3 --warmup 3 --no-e2e --no-cpu-baseline --programs-out gpurun_out/r02_programs_n1.json > gpurun_out/r02_bench_n1_progs.log 2>&1; echo "n1 rc=$?"
ls -la gpurun_out/r02_programs_n*.json
