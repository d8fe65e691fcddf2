#!/usr/bin/env python
"""Launch-shape sweep of the step kernel in local mode (8 slots x 256 MiB
bf16 on one GPU): per program, device time and algorithmic HBM GB/s for each
(threads, unroll, CTAs) combination.
  python tools/tune_local.py [--programs 0,7,200] [--iters 5]"""
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
    ap.add_argument("--programs", default="0,7,200")
    ap.add_argument("--iters", type=int, default=5)
    ap.add_argument("--mib", type=int, default=256)
    args = ap.parse_args()
    import torch
    import bench
    from paper_2110_10548_b200 import executor
    entries = bench.programs()
    elems = (args.mib << 20) // 2
    ctx = executor.Context.local(8, [0] * 8, args.mib << 20)
    for d in range(8):
        ctx.buffer(d, elems, "bf16").normal_()
    stream = torch.cuda.current_stream()
    for i in map(int, args.programs.split(",")):
        prog = entries[i]["prog"]
        plan = ctx.compile(prog, elems, "bf16")
        hbm = sum(plan.step_bytes(s)[1] for s in range(len(prog.steps)))
        for threads, unroll, cps in itertools.product([256, 512], [4, 8], [1, 2, 3, 4]):
            if threads * cps > 2048:
                continue
            plan.set_launch(max_ctas=148 * cps, threads=threads)
            plan.set_option("unroll", unroll)
            for _ in range(2):
                plan.run()
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
            print(json.dumps({"program": i, "text": prog.text[:60], "threads": threads, "unroll": unroll,
                              "ctas": 148 * cps, "us": round(us, 1), "hbm_GBps": round(hbm / (us * 1e-6) / 1e9, 1)}),
                  flush=True)
        plan.close()
    ctx.close()


if __name__ == "__main__":
    main()
