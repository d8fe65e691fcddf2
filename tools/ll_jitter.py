"""Run-to-run spread of a small AllReduce (one-shot path): 30 graph replays
of 20 ops each at 1 KiB / 64 KiB / 256 KiB, max over ranks.
  torchrun --nproc-per-node 4 tools/ll_jitter.py"""
import os, sys, statistics, json
sys.path.insert(0, os.getcwd())
import torch, torch.distributed as dist
from paper_2110_10548_b200 import executor, planner
world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
torch.cuda.set_device(rank); dev = torch.device("cuda", rank)
dist.init_process_group("nccl", device_id=dev)
prog = planner.synthesize(planner.config_path({2:"b200_flat2",4:"b200_sock4"}[world]), [world], [0], payload_bytes=1).placements[0].programs[0]
ctx = executor.Context.from_process_group(world, list(range(world)), 4 << 20)
stream = torch.cuda.current_stream(dev)
res = {}
for nbytes in (1024, 65536, 262144):
    plan = ctx.compile(prog, nbytes // 2, "bf16")
    for _ in range(5): plan.run()
    torch.cuda.synchronize(); dist.barrier()
    g = torch.cuda.CUDAGraph(); s = torch.cuda.Stream(dev); s.wait_stream(stream)
    with torch.cuda.stream(s):
        with torch.cuda.graph(g, stream=s):
            for _ in range(20): plan.run()
    torch.cuda.synchronize(); dist.barrier()
    samples = []
    for trial in range(30):
        dist.barrier()
        a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
        a.record(stream); g.replay(); b.record(stream); torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) * 1e3 / 20], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        samples.append(round(float(t.item()), 2))
    res[nbytes] = samples
    del g; plan.close()
if rank == 0:
    for k, v in res.items():
        print(k, "median", statistics.median(v), "min", min(v), "max", max(v), "n>1.5x median:", sum(x > 1.5 * statistics.median(v) for x in v), v[:12], flush=True)
dist.barrier(); ctx.close(); dist.destroy_process_group()
