# Final 1-GPU evidence: suite, smoke, bench + reference arm (the driver's commands), then ncu of the bench command.
set -x
timeout 1800 python -m pytest tests -m gpu -v -rs > gpurun_out/r02c_pytest_gpu_1.log 2>&1; echo "pytest rc=$?"; tail -2 gpurun_out/r02_pytest_gpu_1_final.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02c_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r02c_bench_n1.log 2>&1; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r02c_ref_n1.log 2>&1; echo "ref rc=$?"
timeout 900 python bench.py --workload config3 --steps 10 --warmup 3 --no-e2e > gpurun_out/r02c_bench_c3_n1.log 2>&1; echo "c3 rc=$?"
for f in r02c_bench_n1 r02c_ref_n1 r02c_bench_c3_n1; do python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], (d.get('roofline') or {}).get('frac'), (d.get('e2e') or {}).get('value'), (d.get('clocks') or {}).get('sm_mhz'), (d.get('cpu_baseline') or {}).get('value'))" gpurun_out/$f.log; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all"
$CMD > gpurun_out/r02c_ncu_plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 3000 --csv --log-file gpurun_out/r02c_launches_n1.csv $CMD > gpurun_out/r02c_ncu_launches.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:StepKernel -s 6 -c 3 -o gpurun_out/r02c_prof_n1 $CMD > gpurun_out/r02c_ncu_full.log 2>&1
echo "ncu rc=$?"
# piece_queue=2 (queue in multi-rank pull phases too) through the emulated-rank suite
RS_PIECE_QUEUE=2 timeout 1200 python -m pytest tests/test_gpu_emulated_ranks.py -q -x > gpurun_out/r02c_emul_pq2.log 2>&1; echo "emul pq2 rc=$?"; tail -1 gpurun_out/r02c_emul_pq2.log
