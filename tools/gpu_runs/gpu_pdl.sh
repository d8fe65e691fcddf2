# PDL A/B at N=1 (config 2 and 3), then the full 1-GPU suite with PDL on.
set -x
for P in 1 0; do
RS_PDL=$P timeout 900 python bench.py --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pdl${P}_c2.log 2>&1; echo "c2 pdl=$P rc=$?"
python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_pdl${P}_c2.log
RS_PDL=$P timeout 900 python bench.py --workload config3 --steps 5 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all > gpurun_out/r02_pdl${P}_c3.log 2>&1; echo "c3 pdl=$P rc=$?"
python -c "
import json,sys
for l in open(sys.argv[1]):
    if l.startswith('{'): d=json.loads(l); print(d['value'], d['ms_per_step'], d['roofline']['frac'])" gpurun_out/r02_pdl${P}_c3.log
done
timeout 1800 python -m pytest tests -m gpu -v -rs > gpurun_out/r02_pytest_gpu_1_pdl.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/r02_pytest_gpu_1_pdl.log
