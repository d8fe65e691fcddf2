#!/usr/bin/env python
"""Placement effect on NVSwitch + simulator rescoring (BASELINE configs 3/5).

One slot per GPU (K = N). For each request (descriptor, axes, reduction axes)
every placement's every synthesized program is timed on the GPUs (device
time, an untimed run absorbs rank skew, then 2 timed back-to-back runs, max
over ranks) next to the reference cost model's prediction (`Simulate`,
simulator.cc:141-188, with the descriptor's 900 GB/s levels). Reports, per
placement, the baseline AllReduce and the best program measured vs predicted,
and the simulator's top-k accuracy over all (placement, request) instances.

  torchrun --nproc-per-node 4 tools/placement_study.py --out profiles/placement_n4.json
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

REQUESTS = {
    4: [("b200_sock4", [2, 2], [0]), ("b200_sock4", [2, 2], [1]), ("b200_sock4", [4], [0]),
        ("b200_flat4", [2, 2], [0]), ("b200_flat4", [4], [0])],
    2: [("b200_flat2", [2], [0])],
    8: [("b200_sock", [2, 4], [0]), ("b200_sock", [2, 4], [1]), ("b200_sock", [2, 4], [0, 1]),
        ("b200_sock", [2, 2, 2], [0]), ("b200_sock", [2, 2, 2], [0, 2]), ("b200_flat8", [8], [0])],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--out", default=None)
    ap.add_argument("--max-programs", type=int, default=300)
    args = ap.parse_args()
    import torch
    import torch.distributed as dist
    from paper_2110_10548_b200 import executor, planner, rescore
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    es = 2 if args.dtype == "bf16" else 4
    nbytes = args.mib << 20
    K = world
    ctx = executor.Context.from_process_group(K, list(range(K)), nbytes)
    ctx.buffer(rank, nbytes // es, args.dtype).normal_()
    stream = torch.cuda.current_stream(dev)
    rows, placements = [], []
    for desc, axes, red in REQUESTS[world]:
        syn = planner.synthesize(planner.config_path(desc), axes, red, payload_bytes=nbytes)
        for mi, pl in enumerate(syn.placements):
            times = []
            for pi, prog in enumerate(pl.programs[: args.max_programs]):
                plan = ctx.compile(prog, nbytes // es, args.dtype)
                plan.run()
                a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                a.record(stream)
                plan.run()
                plan.run()
                b.record(stream)
                torch.cuda.synchronize()
                t = torch.tensor([a.elapsed_time(b) * 1e3 / 2], device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                us = float(t.item())
                plan.close()
                times.append(us)
                rows.append({"instance": f"{desc}|{axes}|{red}|{mi}", "index": pi, "sim_seconds": prog.seconds,
                             "measured_us": us, "text": prog.text})
            best = min(range(len(times)), key=lambda i: times[i])
            sim_best = min(range(len(times)), key=lambda i: (pl.programs[i].seconds, i))
            placements.append({"descriptor": desc, "axes": axes, "reduce": red, "matrix": mi,
                               "factors": pl.factors, "partition": pl.partition, "programs": len(times),
                               "allreduce_us": times[0], "allreduce_sim_us": pl.programs[0].seconds * 1e6,
                               "best_us": times[best], "best": pl.programs[best].text,
                               "sim_best": pl.programs[sim_best].text, "sim_best_us": times[sim_best],
                               "sim_best_predicted_us": pl.programs[sim_best].seconds * 1e6})
            if rank == 0:
                print(json.dumps(placements[-1]), flush=True)
    summary = rescore.topk(rows)
    if rank == 0:
        print(json.dumps({"top_k": summary["top_k"], "top_k_tie_aware": summary["top_k_tie_aware"],
                          "instances": summary["instances"]}), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump({"world": world, "mib": args.mib, "dtype": args.dtype, "nvls": ctx.nvls,
                           "placements": placements, "rescoring": summary, "programs": rows}, f)
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
