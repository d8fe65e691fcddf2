#!/usr/bin/env python
"""One-shot vs pull for groups with several members per GPU: config-2
AllReduce program (8 slots) on 2 or 4 GPUs in one process, small sizes,
device time per run from rs_plan_time (slowest GPU).
  python tools/ll_colocated.py [--gpus 2]"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    args = ap.parse_args()
    import bench
    from paper_2110_10548_b200 import executor
    n = args.gpus
    entries = bench.programs()
    ctx = executor.Context.local(8, [d * n // 8 for d in range(8)], 4 << 20)
    for idx in (0, 7):
        prog = entries[idx]["prog"]
        for nbytes in (1 << 10, 8 << 10, 64 << 10, 256 << 10, 1 << 20):
            row = {}
            for ll in (0, 256 << 10):
                ctx.set_option("ll_max_bytes", ll)
                ctx.set_option("ll_total_bytes", 3 << 20)
                plan = ctx.compile(prog, nbytes // 2, "bf16")
                row["one-shot" if ll else "pull"] = round(plan.time_us(3, 50), 2)
                row["ll_phases" if ll else "_"] = sum(plan.describe()["phase_ll"]) if ll else None
                plan.close()
            print(idx, prog.text[:50], nbytes, row, flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
