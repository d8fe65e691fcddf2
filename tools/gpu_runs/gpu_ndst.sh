python tools/local_ops.py > gpurun_out/r02_lo_ndst.log 2>&1; cat gpurun_out/r02_lo_ndst.log
for i in 1 2; do timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_bench_ndst_$i.log 2>&1; python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_bench_ndst_$i.log; done
