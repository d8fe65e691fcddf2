for V in 2 0 2 0; do RS_VEC256=$V timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_bench_v256b_$V.log 2>&1; python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_bench_v256b_$V.log; done
for V in 2 0; do RS_VEC256=$V timeout 900 python bench.py --workload config3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_bench_c3_v256_$V.log 2>&1; python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_bench_c3_v256_$V.log; done
