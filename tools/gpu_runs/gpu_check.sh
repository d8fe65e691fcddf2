set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_ranks_one_gpu.py -x -q -s > gpurun_out/r02_pytest_ranks1gpu.log 2>&1; echo "ranks rc=$?"
tail -5 gpurun_out/r02_pytest_ranks1gpu.log
timeout 900 python -m pytest tests -m gpu -q --deselect tests/test_gpu_ranks_one_gpu.py > gpurun_out/r02_pytest_gpu_1.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/r02_pytest_gpu_1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 5 --warmup 3 > gpurun_out/r02_bench_n1.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/r02_bench_n1.log
timeout 600 python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r02_ref_n1.log 2>&1; echo "ref rc=$?"
tail -c 1500 gpurun_out/r02_ref_n1.log
