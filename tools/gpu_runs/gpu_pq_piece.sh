# With the piece queue: local piece size A/B (RS_MAX_PIECE) per op and on the N=1 bench.
for P in 65536 32768 131072 262144 65536; do echo "max_piece=$P"; RS_MAX_PIECE=$P python tools/local_ops.py 2>&1 | cut -c1-75; done
for P in 65536 131072 65536 131072; do
  RS_MAX_PIECE=$P python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pp_$P.log 2>&1
  python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['roofline']['frac'])" gpurun_out/r02_pp_$P.log
done
