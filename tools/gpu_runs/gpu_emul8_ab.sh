# Emulated N=8 bench path: which final-code change moves it (piece_queue 2 vs 1, wave_lag 2 vs 0).
for cfg in "2 2" "1 2" "2 0" "1 0"; do
  set -- $cfg
  RS_PIECE_QUEUE=$1 RS_WAVE_LAG=$2 timeout 600 python bench.py --emulate-ranks 8 --steps 2 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_emu8_q$1_l$2.log 2>&1
  python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'):
        d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'])" gpurun_out/r02_emu8_q$1_l$2.log
done
