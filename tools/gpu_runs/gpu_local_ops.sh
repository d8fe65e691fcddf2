# Local-mode per-op HBM efficiency: default vs wide loads vs unroll/threads variants; quick parity with wide loads.
set -x
python tools/local_ops.py > gpurun_out/r02_local_ops_base.log 2>&1; cat gpurun_out/r02_local_ops_base.log
python tools/local_ops.py --opt local_wide=1 > gpurun_out/r02_local_ops_wide.log 2>&1; cat gpurun_out/r02_local_ops_wide.log
python tools/local_ops.py --opt threads=256 > gpurun_out/r02_local_ops_t256.log 2>&1; cat gpurun_out/r02_local_ops_t256.log
python tools/local_ops.py --opt max_ctas=296 --opt threads=256 > gpurun_out/r02_local_ops_t256c296.log 2>&1; cat gpurun_out/r02_local_ops_t256c296.log
RS_LOCAL_WIDE=1 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -x -k "local or ragged or repeated or graph" > gpurun_out/r02_local_wide_parity.log 2>&1; echo "parity rc=$?"; tail -2 gpurun_out/r02_local_wide_parity.log
