# Verify the local_dynamic gain: full-size parity, per-op A/B, ncu DRAM bytes of the same launches.
RS_LOCAL_DYNAMIC=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "local or full_size or ragged or repeated or graph or user or upload" > gpurun_out/r02_ldyn2_parity.log 2>&1; echo "parity rc=$?"; tail -1 gpurun_out/r02_ldyn2_parity.log
for D in 0 1; do echo "local_dynamic=$D"; RS_LOCAL_DYNAMIC=$D python tools/local_ops.py 2>&1 | cut -c1-90; done
CMD="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu-baseline --no-rescore-all"
RS_LOCAL_DYNAMIC=1 $CMD > gpurun_out/r02c_ncu_plain.log 2>&1 && \
RS_LOCAL_DYNAMIC=1 ncu --set full --clock-control none --import-source on -k regex:StepKernel -s 6 -c 3 -o gpurun_out/r02c_prof_n1 $CMD > gpurun_out/r02c_ncu_full.log 2>&1
echo "ncu rc=$?"
