for D in 1 0 1 0; do RS_LOCAL_DYNAMIC=$D timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_ldyn_$D.log 2>&1; python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(sys.argv[1], d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_ldyn_$D.log; done
RS_LOCAL_DYNAMIC=1 timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "local or ragged or repeated or graph" > gpurun_out/r02_ldyn_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02_ldyn_parity.log
