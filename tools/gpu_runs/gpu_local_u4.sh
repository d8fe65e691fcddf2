python tools/local_ops.py > gpurun_out/r02_lo_u8.log 2>&1; cat gpurun_out/r02_lo_u8.log
python tools/local_ops.py --opt unroll=4 > gpurun_out/r02_lo_u4.log 2>&1; cat gpurun_out/r02_lo_u4.log
python tools/local_ops.py --opt unroll=4 --opt max_ctas=444 > gpurun_out/r02_lo_u4c444.log 2>&1; cat gpurun_out/r02_lo_u4c444.log
