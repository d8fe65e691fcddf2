# Last check of the final code on one GPU: GPU suite, smoke, emulated N=8 bench path.
timeout 1500 python -m pytest tests -m gpu -q -rs > gpurun_out/r02i_pytest_gpu_1.log 2>&1; echo "pytest rc=$?"; tail -1 gpurun_out/r02i_pytest_gpu_1.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02i_smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r02i_smoke.log
timeout 600 python bench.py --emulate-ranks 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02i_bench_emulated8.log 2>&1; echo "emu8 rc=$?"
python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['ms_per_step'])" gpurun_out/r02i_bench_emulated8.log
