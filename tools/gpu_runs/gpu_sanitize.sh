# compute-sanitizer (memcheck, racecheck, synccheck) on the local path and on two ranks over IPC on cuda:0.
set -x
CS=/usr/local/cuda/bin/compute-sanitizer
K="--kernel-name regex:StepKernel|NvlsSelfCheck --print-limit 50"
for tool in memcheck racecheck synccheck; do
  timeout 1200 $CS --tool $tool $K python tools/sanitize_run.py > gpurun_out/r02_sanitizer_${tool}_local.txt 2>&1; echo "$tool local rc=$?"; tail -4 gpurun_out/r02_sanitizer_${tool}_local.txt
  timeout 1500 $CS --tool $tool --target-processes all $K python tools/sanitize_run.py --world 2 > gpurun_out/r02_sanitizer_${tool}_world2.txt 2>&1; echo "$tool world2 rc=$?"; tail -4 gpurun_out/r02_sanitizer_${tool}_world2.txt
done
python tools/hbm_probe.py > gpurun_out/r02_hbm_probe.txt 2>&1; cat gpurun_out/r02_hbm_probe.txt
