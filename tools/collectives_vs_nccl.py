#!/usr/bin/env python
"""Single-step programs against NCCL's matching collective, one slot per GPU
(graph mode, max over ranks): AllReduce vs all_reduce, ReduceScatter vs
reduce_scatter_tensor, Reduce (root 0) vs reduce. Bytes = per-GPU buffer.
  torchrun --nproc-per-node 4 tools/collectives_vs_nccl.py [--out f.json]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--min-bytes", type=int, default=1 << 12)
    ap.add_argument("--max-bytes", type=int, default=1 << 30)
    ap.add_argument("--step", type=int, default=8)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--out", default=None)
    ap.add_argument("--ops", default="AllReduce,ReduceScatter,Reduce")
    ap.add_argument("--reduce-modes", default="0",
                    help="comma list of executor Reduce variants to time (0 pull, 1 push, 2 NVLS, 3 NVLS root)")
    ap.add_argument("--nvls", action="store_true", help="multicast-capable heaps (RS_NVLS=1; needed by modes 2/3)")
    ap.add_argument("--push-min-bytes", type=int, default=None, help="context push threshold (-1 = never push)")
    ap.add_argument("--wave-bytes", type=int, default=None, help="push waves (0 = one wave)")
    ap.add_argument("--ll-max-bytes", type=int, default=None, help="one-shot budget (0 = never one-shot)")
    ap.add_argument("--reduce-wave-bytes", type=int, default=None, help="Reduce push waves")
    ap.add_argument("--bcast-nvls", type=int, default=0, help="with --nvls: Broadcast by multicast stores")
    args = ap.parse_args()
    if args.nvls:
        os.environ["RS_NVLS"] = "1"
    import torch
    import torch.distributed as dist
    from paper_2110_10548_b200 import executor
    from paper_2110_10548_b200.planner import LoweredProgram
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("nccl", device_id=dev)
    stream = torch.cuda.current_stream(dev)
    ctx = executor.Context.from_process_group(world, list(range(world)), args.max_bytes)
    if args.push_min_bytes is not None:
        ctx.set_option("push_min_bytes", args.push_min_bytes)
    if args.wave_bytes is not None:
        ctx.set_option("push_wave_bytes", args.wave_bytes)
    if args.ll_max_bytes is not None:
        ctx.set_option("ll_max_bytes", args.ll_max_bytes)
    if args.reduce_wave_bytes is not None:
        ctx.set_option("reduce_wave_bytes", args.reduce_wave_bytes)
    g = list(range(world))
    ops = args.ops.split(",")
    modes = [int(m) for m in args.reduce_modes.split(",")]
    progs = {"AllReduce": LoweredProgram(steps=[(0, [g])]), "ReduceScatter": LoweredProgram(steps=[(1, [g])]),
             "Reduce": LoweredProgram(steps=[(3, [g])]),
             # Reduce then Broadcast (a Broadcast needs a step that empties members first)
             "ReduceBroadcast": LoweredProgram(steps=[(3, [g]), (4, [g])])}
    progs = {k: v for k, v in progs.items() if k in ops}

    def timed(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        dist.barrier()
        graph = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream(dev)
        s.wait_stream(stream)
        with torch.cuda.stream(s):
            with torch.cuda.graph(graph, stream=s):
                for _ in range(args.iters):
                    fn()
        torch.cuda.synchronize()
        dist.barrier()
        graph.replay()
        torch.cuda.synchronize()
        dist.barrier()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        graph.replay()
        b.record(stream)
        torch.cuda.synchronize()
        t = torch.tensor([a.elapsed_time(b) * 1e3 / args.iters], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        del graph
        return float(t.item())

    rows = []
    size = args.min_bytes
    while size <= args.max_bytes:
        elems = size // 2
        x = torch.randn(elems, device=dev).to(torch.bfloat16)
        out = torch.empty(elems // world, device=dev, dtype=torch.bfloat16)
        nccl = {"AllReduce": lambda: dist.all_reduce(x),
                "ReduceScatter": lambda: dist.reduce_scatter_tensor(out, x),
                "Reduce": lambda: dist.reduce(x, dst=0),
                "ReduceBroadcast": lambda: (dist.reduce(x, dst=0), dist.broadcast(x, src=0))}
        row = {"bytes": size}
        for name, prog in progs.items():
            theirs = timed(nccl[name])
            for mode in (modes if name == "Reduce" else [None]):
                if mode is not None:
                    ctx.set_option("reduce_mode", mode)
                if args.nvls:  # NVLS only where a Reduce mode or --bcast-nvls asks for it
                    bc = name == "ReduceBroadcast" and args.bcast_nvls
                    ctx.set_option("nvls_min_bytes", 0 if (mode in (2, 3) or bc) else -1)
                    ctx.set_option("nvls_bcast", 1 if bc else 0)
                plan = ctx.compile(prog, elems, "bf16")
                ours = timed(plan.run)
                used = sorted({t["mode"] for st in plan.describe()["steps"] for rk in st["ranks"] for t in rk["tasks"]})
                plan.close()
                key = name if mode is None else f"{name}[mode {mode}]"
                row[key] = {"ours_us": round(ours, 2), "nccl_us": round(theirs, 2), "speedup": round(theirs / ours, 3),
                            "task_modes": used}
        rows.append(row)
        if rank == 0:
            print(json.dumps(row), flush=True)
        size *= args.step
    if rank == 0 and args.out:
        json.dump({"K": world, "rows": rows}, open(args.out, "w"))
    dist.barrier()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
