#!/usr/bin/env python
"""Config 4 of BASELINE.json: message-size sweep at K = N GPUs (one program
device per GPU), every synthesized program of the K-GPU descriptor against
NCCL's default AllReduce on the same bytes.

  torchrun --nproc-per-node N bench_sweep.py [--dtype bf16] [--min-bytes 1024]
           [--max 1073741824] [--iters 20] [--out profiles/sweep_nN.json]

Descriptors: K=2 [(node,1),(gpu,2)]; K=4 [(node,1),(socket,2),(gpu,2)];
K=8 [(node,1),(socket,2),(gpu,4)] axes [8].
Times are device times (CUDA events, median of --iters after warm-up), max
over ranks. Bus GB/s = (D / T) * 2(n-1)/n (nccl-tests AllReduce convention).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

DESCRIPTORS = {2: "b200_flat2", 4: "b200_sock4", 8: "b200_sock"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--min-bytes", dest="min", type=int, default=1 << 10)
    ap.add_argument("--max-bytes", dest="max", type=int, default=1 << 30)
    ap.add_argument("--iters", type=int, default=20)
    ap.add_argument("--step", type=int, default=2, help="size multiplier between rows")
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--programs", default="all", help="'all' or 'first:N'")
    ap.add_argument("--out", default=None)
    ap.add_argument("--graph", action="store_true",
                    help="time `iters` back-to-back ops captured in one CUDA graph (both arms)")
    ap.add_argument("--no-nvls", action="store_true", help="P2P kernels only (bit-exact everywhere)")
    args = ap.parse_args()
    if not args.no_nvls:
        os.environ.setdefault("RS_NVLS", "1")  # AllReduce groups of >= 4 GPUs at >= 16 MiB

    import torch
    import torch.distributed as dist

    from paper_2110_10548_b200 import executor, planner

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ.get("LOCAL_RANK", rank))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    K = world
    syn = planner.synthesize(planner.config_path(DESCRIPTORS[K]), [K], [0], payload_bytes=1)
    progs = syn.placements[0].programs
    if args.programs.startswith("first:"):
        progs = progs[: int(args.programs.split(":")[1])]
    es = 2 if args.dtype == "bf16" else 4
    tdtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    ctx = executor.Context.from_process_group(K, list(range(K)), args.max)
    buf = ctx.buffer(rank, args.max // es, args.dtype)
    buf.normal_()
    nccl_buf = torch.randn(args.max // es, device=dev).to(tdtype)
    stream = torch.cuda.current_stream(dev)

    def timed(fn):
        for _ in range(args.warmup):
            fn()
        dist.barrier()
        torch.cuda.synchronize()
        times = []
        for _ in range(args.iters):
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            times.append((a, b))
        torch.cuda.synchronize()
        us = statistics.median(a.elapsed_time(b) * 1e3 for a, b in times)
        t = torch.tensor([us], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    if args.graph:
        eager_timed = timed

        def timed(fn):  # noqa: F811 — per-op device time from a graph of `iters` back-to-back ops
            for _ in range(args.warmup):
                fn()
            torch.cuda.synchronize()
            dist.barrier()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream(device=dev)
            s.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    for _ in range(args.iters):
                        fn()
            torch.cuda.synchronize()
            dist.barrier()
            g.replay()  # warm replay
            torch.cuda.synchronize()
            dist.barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            g.replay()
            b.record(stream)
            torch.cuda.synchronize()
            us = a.elapsed_time(b) * 1e3 / args.iters
            t = torch.tensor([us], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            del g
            return float(t.item())

        del eager_timed

    results = []
    size = args.min
    while size <= args.max:
        elems = size // es
        row = {"bytes": size, "nccl_us": None, "programs": []}
        x = nccl_buf[:elems]
        row["nccl_us"] = timed(lambda: dist.all_reduce(x))
        for p in progs:
            plan = ctx.compile(p, elems, args.dtype)
            us = timed(plan.run)
            row["programs"].append({"text": p.text, "us": us, "sim_s": p.seconds})
            plan.close()
        best = min(row["programs"], key=lambda r: r["us"])
        f = 2.0 * (K - 1) / K
        row["best"] = best["text"]
        row["best_us"] = best["us"]
        row["best_busbw"] = size / (best["us"] * 1e-6) * f / 1e9
        row["nccl_busbw"] = size / (row["nccl_us"] * 1e-6) * f / 1e9
        row["speedup_vs_nccl"] = row["nccl_us"] / best["us"]
        ar = row["programs"][0]
        row["allreduce_program_us"] = ar["us"]
        results.append(row)
        if rank == 0:
            print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in row.items()
                              if k != "programs"}), flush=True)
        size *= args.step
    if rank == 0 and args.out:
        with open(args.out, "w") as f:
            json.dump({"K": K, "dtype": args.dtype, "descriptor": DESCRIPTORS[K], "rows": results}, f)
    dist.barrier()
    del buf
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
