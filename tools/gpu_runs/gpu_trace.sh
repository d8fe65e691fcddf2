# Piece timelines (profiling build) of cross-GPU steps at K=4.
set -x
export RS_BARRIER_TIMEOUT_S=20
make -s profiling >/dev/null 2>&1 || true
run() { name=$1; shift; timeout 300 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 29541 tools/trace_push.py "$@" --out gpurun_out/r02_trace_$name.json > gpurun_out/r02_trace_$name.log 2>&1; echo "$name rc=$?"; cat gpurun_out/r02_trace_$name.log | grep -v Warning; }
run red1g_m1w16 --op reduce --mib 1024 --reduce-mode 1 --wave-mib 16
run red1g_m0 --op reduce --mib 1024 --reduce-mode 0
run ar1g_push --op allreduce --mib 1024
run ar64_push --op allreduce --mib 64
run red64_m1w4 --op reduce --mib 64 --reduce-mode 1 --wave-mib 4
run red64_m0 --op reduce --mib 64 --reduce-mode 0
