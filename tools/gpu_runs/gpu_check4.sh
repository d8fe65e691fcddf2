# 4-GPU lease: full GPU suite log, Reduce variant A/B vs NCCL, collectives, N=8 dry run.
set -x
nvidia-smi topo -m | head -8
mkdir -p gpurun_out
export RS_BARRIER_TIMEOUT_S=20
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r02_pytest_gpu_4.log 2>&1; echo "pytest rc=$?"
tail -8 gpurun_out/r02_pytest_gpu_4.log
timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29511 tools/collectives_vs_nccl.py --ops Reduce --reduce-modes 0,1,2,3 --nvls --min-bytes 1048576 --max-bytes 1073741824 --step 4 --out gpurun_out/r02_reduce_modes_k4.json > gpurun_out/r02_reduce_modes_k4.log 2>&1; echo "reduce rc=$?"
cat gpurun_out/r02_reduce_modes_k4.log | grep bytes
timeout 900 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29512 tools/collectives_vs_nccl.py --ops AllReduce,ReduceScatter --out gpurun_out/r02_collectives_k4.json > gpurun_out/r02_collectives_k4.log 2>&1; echo "coll rc=$?"
cat gpurun_out/r02_collectives_k4.log | grep bytes
timeout 1200 torchrun --nnodes=1 --nproc-per-node 8 --master-addr 127.0.0.1 --master-port 29513 bench.py --gpus 8 --ranks-per-gpu 2 --steps 1 --warmup 3 --no-e2e > gpurun_out/r02_bench_dryrun_n8_on4.log 2>&1; echo "dry rc=$?"
tail -c 2500 gpurun_out/r02_bench_dryrun_n8_on4.log
