# Final code: the N=8 bench code path (one slot per rank, 8 ranks) emulated on one GPU; not a performance number.
timeout 900 python bench.py --emulate-ranks 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/r02h_bench_emulated8.log 2>&1; echo "emu8 rc=$?"
python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['bound'], d['config']['parallelism'], d.get('simulator_rescoring',{}).get('instances'))" gpurun_out/r02h_bench_emulated8.log
