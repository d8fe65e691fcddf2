# What the driver runs at round end on one GPU: GPU suite, smoke, bench, reference arm.
set -x
timeout 1800 python -m pytest tests -m gpu -v -rs --durations=10 > gpurun_out/r02_pytest_gpu_1_final.log 2>&1; echo "pytest rc=$?"; tail -18 gpurun_out/r02_pytest_gpu_1_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02_smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/r02_smoke.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02_bench_n1_final.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02_ref_n1_final.log 2>&1; echo "ref rc=$?"
for f in r02_bench_n1_final r02_ref_n1_final; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), d.get('clocks'), (d.get('cpu_baseline') or {}).get('value'))" gpurun_out/$f.log; done
python tools/hbm_probe.py > gpurun_out/r02_hbm_probe.txt 2>&1; cat gpurun_out/r02_hbm_probe.txt
