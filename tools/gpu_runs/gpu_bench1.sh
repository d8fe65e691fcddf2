# 1-GPU: bench config 2 (default) and config 3, reference arm.
set -x
timeout 1200 python bench.py --steps 5 --warmup 3 --programs-out gpurun_out/r02_programs_n1.json > gpurun_out/r02_bench_n1.log 2>&1; echo "bench rc=$?"
tail -c 4000 gpurun_out/r02_bench_n1.log
timeout 1200 python bench.py --workload config3 --steps 5 --warmup 3 --no-e2e > gpurun_out/r02_bench_c3_n1.log 2>&1; echo "bench c3 rc=$?"
tail -c 3000 gpurun_out/r02_bench_c3_n1.log
