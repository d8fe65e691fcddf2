#!/usr/bin/env python
"""Launch-knob sweep of the step kernel over NVLink (one rank per GPU).
  torchrun --nproc-per-node N tools/tune_nvlink.py [--mib 256] [--program 0]
Prints bus GB/s of the chosen K=N program for each (threads, unroll, ctas)."""
import argparse
import itertools
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--program", type=int, default=0)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--push", type=int, default=-1, help="1 = push variant, 0 = pull, -1 = default threshold")
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2110_10548_b200 import executor, planner
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    desc = {2: "b200_flat2", 4: "b200_flat4", 8: "b200_flat8"}[world]
    prog = planner.synthesize(planner.config_path(desc), [world], [0]).placements[0].programs[args.program]
    es = 2 if args.dtype == "bf16" else 4
    nbytes = args.mib << 20
    ctx = executor.Context.from_process_group(world, list(range(world)), nbytes)
    if args.push >= 0:
        ctx.set_option("push_min_bytes", 0 if args.push else -1)
    ctx.buffer(rank, nbytes // es, args.dtype).normal_()
    plan = ctx.compile(prog, nbytes // es, args.dtype)
    stream = torch.cuda.current_stream(dev)
    f = 2.0 * (world - 1) / world
    rows = []
    for threads, unroll, cps in itertools.product([256, 512], [4, 8], [1, 2, 4]):
        if threads * cps > 2048:
            continue
        plan.set_launch(max_ctas=148 * cps, threads=threads)
        plan.set_option("unroll", unroll)
        for _ in range(3):
            plan.run()
        dist.barrier()
        torch.cuda.synchronize()
        evs = []
        for _ in range(args.iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            plan.run()
            b.record(stream)
            evs.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median(a.elapsed_time(b) * 1e3 for a, b in evs)
        t = torch.tensor([us], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        us = float(t.item())
        row = {"threads": threads, "unroll": unroll, "ctas": 148 * cps, "us": round(us, 1),
               "busbw": round(nbytes / (us * 1e-6) * f / 1e9, 1)}
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
    ctx.synchronize()
    plan.close()
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
