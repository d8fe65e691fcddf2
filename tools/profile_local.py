#!/usr/bin/env python
"""Small single-GPU driver for ncu captures (never run ncu on a multi-rank
command): config-2 programs at full size (8 slots x 256 MiB bf16) in local
mode. `--programs i,j,...` selects programs by index in bench.py's order."""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--programs", default="0,7,200")
    ap.add_argument("--repeat", type=int, default=3)
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
    for i in map(int, args.programs.split(",")):
        plan = ctx.compile(entries[i]["prog"], elems, "bf16")
        for _ in range(args.repeat):
            plan.run()
        torch.cuda.synchronize()
        print(i, entries[i]["prog"].text, flush=True)
        plan.close()
    ctx.synchronize()
    ctx.close()


if __name__ == "__main__":
    main()
