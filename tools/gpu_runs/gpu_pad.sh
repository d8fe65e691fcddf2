# Slot padding A/B (DRAM interleaving of slots a power of two apart) and a single-group broadcast.
for P in 0 1 3 0; do echo "pad=$P"; RS_SLOT_PAD_MIB=$P python tools/local_ops.py 2>&1 | cut -c1-90; done
for P in 1 0; do RS_SLOT_PAD_MIB=$P timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pad_$P.log 2>&1; python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_pad_$P.log; done
