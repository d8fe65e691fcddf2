set -x
timeout 1800 python -m pytest tests -m gpu -v -rs > gpurun_out/r02h_pytest_gpu_1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_gpu_1_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02h_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02h_bench_n1.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02h_ref_n1.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --workload config3 --steps 10 --warmup 3 --no-e2e > gpurun_out/r02h_bench_c3_n1.log 2>&1; echo "c3 rc=$?"
for f in r02h_bench_n1 r02h_ref_n1 r02h_bench_c3_n1; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('cpu_baseline') or {}).get('value'))" gpurun_out/$f.log; done
# piece_queue=2 (queue in multi-rank pull phases too) through the emulated-rank suite
