# One-GPU launch-shape A/B with 256-bit vectors: pieces 64/128/256 KiB, unroll 4 (2 CTAs/SM) vs 8.
python tools/local_ops.py > gpurun_out/r02_ls_base.log 2>&1; echo base; cat gpurun_out/r02_ls_base.log | cut -c1-90
RS_MAX_PIECE=131072 python tools/local_ops.py > gpurun_out/r02_ls_p128.log 2>&1; echo p128; cat gpurun_out/r02_ls_p128.log | cut -c1-90
RS_MAX_PIECE=262144 python tools/local_ops.py > gpurun_out/r02_ls_p256.log 2>&1; echo p256; cat gpurun_out/r02_ls_p256.log | cut -c1-90
python tools/local_ops.py --opt unroll=4 > gpurun_out/r02_ls_u4.log 2>&1; echo u4; cat gpurun_out/r02_ls_u4.log | cut -c1-90
