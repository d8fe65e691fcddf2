#!/usr/bin/env python
"""Per-collective HBM efficiency of the step kernel in local mode (8 slots x
256 MiB bf16 on one GPU, the bench's N=1 shape): single-step and two-step
programs over the config-2 reduction groups {0,1,4,5} {2,3,6,7}, device time
(rs_plan_time) and algorithmic HBM GB/s per program, with plan options given
on the command line (A/B of kernel variants).
  python tools/local_ops.py [--opt local_wide=1] [--opt unroll=4]"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

G = [[0, 1, 4, 5], [2, 3, 6, 7]]
PAIRS = [[0, 1], [2, 3], [4, 5], [6, 7]]
PROGRAMS = {
    "AllReduce": [(0, G)],
    "ReduceScatter": [(1, G)],
    "Reduce": [(3, G)],
    "Reduce+Broadcast": [(3, G), (4, G)],
    "Reduce+AllGather": [(3, G), (2, G)],
    "ReduceScatter+AllGather": [(1, G), (2, G)],
    "AllReduce pairs": [(0, PAIRS)],
    "Reduce pairs+Broadcast": [(3, PAIRS), (4, PAIRS)],
}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--iters", type=int, default=10)
    ap.add_argument("--opt", action="append", default=[], help="plan option key=value")
    args = ap.parse_args()
    import torch
    from paper_2110_10548_b200 import executor
    from paper_2110_10548_b200.planner import LoweredProgram
    elems = (args.mib << 20) // 2
    ctx = executor.Context.local(8, [0] * 8, args.mib << 20)
    for d in range(8):
        ctx.buffer(d, elems, "bf16").normal_()
    torch.cuda.synchronize()
    out = {}
    for name, steps in PROGRAMS.items():
        prog = LoweredProgram(steps=steps)
        plan = ctx.compile(prog, elems, "bf16")
        for kv in args.opt:
            k, v = kv.split("=")
            plan.set_option(k, int(v))
        hbm = [plan.step_bytes(s)[1] for s in range(len(steps))]
        us = plan.time_us(warmup=2, iters=args.iters)
        out[name] = {"us": round(us, 1), "hbm_GB": round(sum(hbm) / 1e9, 3),
                     "GBps": round(sum(hbm) / (us * 1e-6) / 1e9, 1)}
        print(json.dumps({"program": name, **out[name], "opts": args.opt}), flush=True)
        plan.close()
    ctx.close()


if __name__ == "__main__":
    main()
