# 256-bit local vectors: per-op A/B, bench A/B, parity with sums on the 256-bit path.
set -x
for V in 0 1 2; do python tools/local_ops.py --opt vec256=$V > gpurun_out/r02_lo_v256_$V.log 2>&1; cat gpurun_out/r02_lo_v256_$V.log; done
for V in 1 2 0; do RS_VEC256=$V timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_bench_v256_$V.log 2>&1; python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_bench_v256_$V.log; done
RS_VEC256=2 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "local or ragged or repeated or graph or user or upload" > gpurun_out/r02_v256_parity.log 2>&1; echo "parity2 rc=$?"; tail -2 gpurun_out/r02_v256_parity.log
