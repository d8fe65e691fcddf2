export RS_BARRIER_TIMEOUT_S=30
timeout 900 python -m pytest tests/test_gpu_nvls.py tests/test_gpu_emulated_ranks.py -q -x > gpurun_out/r02_bcast_tests.log 2>&1; echo "tests rc=$?"; tail -2 gpurun_out/r02_bcast_tests.log
for B in 0 1 0 1; do
timeout 600 torchrun --nnodes=1 --nproc-per-node 4 --master-addr 127.0.0.1 --master-port 2979$B tools/collectives_vs_nccl.py --ops ReduceBroadcast,Reduce --nvls --bcast-nvls $B --min-bytes 1048576 --max-bytes 1073741824 --step 4 --iters 10 --out gpurun_out/r02_bcast_$B.json > /dev/null 2>&1; echo "B=$B rc=$?"
python -c "
import json,sys
d=json.load(open(sys.argv[1]))
print(sys.argv[2], ' '.join(f\"{r['bytes']>>20}M:\" + '/'.join(f\"{r[k]['ours_us']:.1f}({r[k]['nccl_us']:.0f})\" for k in r if k!='bytes') for r in d['rows']))" gpurun_out/r02_bcast_$B.json B=$B
done
