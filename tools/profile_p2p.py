#!/usr/bin/env python
"""ncu driver for the cross-GPU step kernel (one process, K GPUs, one slot
per GPU): with RS_SOLO_PROFILE=1 the kernels skip their cross-GPU waits, so
ncu (which serialises launches) can replay each GPU's kernel alone and count
its NVLink bytes (nvltx/nvlrx) next to its DRAM bytes. The data is garbage in
this mode — it only measures traffic. The switch exists only in the
profiling build (`make profiling`), which this script selects itself.

  RS_SOLO_PROFILE=1 ncu --metrics gpu__time_duration.sum,nvltx__bytes.sum,nvlrx__bytes.sum,\
dram__bytes_read.sum,dram__bytes_write.sum python tools/profile_p2p.py --gpus 2
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=2)
    ap.add_argument("--mib", type=int, default=256)
    ap.add_argument("--program", type=int, default=0)
    ap.add_argument("--dtype", default="bf16")
    ap.add_argument("--push", type=int, default=0, help="1: push variant (store-only), 0: pull")
    ap.add_argument("--op", default=None, help="one collective over all GPUs instead of a synthesized program: "
                                               "AllReduce | ReduceScatter | Reduce")
    ap.add_argument("--reduce-mode", type=int, default=None, help="context reduce_mode (-1 auto, 0 pull, 1 push)")
    args = ap.parse_args()
    if os.environ.get("RS_SOLO_PROFILE") != "1":
        raise SystemExit("set RS_SOLO_PROFILE=1 (the kernels would wait for peers ncu never runs)")
    os.environ.setdefault("RS_BARRIER_TIMEOUT_S", "2")
    prof = os.path.join(ROOT, "paper_2110_10548_b200", "_lib", "libredsynth_b200_prof.so")
    if not os.path.exists(prof):
        raise SystemExit("build the profiling library first: make profiling")
    os.environ["RS_LIB_PATH"] = prof
    import torch
    from paper_2110_10548_b200 import executor, planner
    n = args.gpus
    desc = {2: "b200_flat2", 4: "b200_flat4", 8: "b200_flat8"}[n]
    if args.op:
        g = list(range(n))
        prog = planner.LoweredProgram(steps=[({"AllReduce": 0, "ReduceScatter": 1, "Reduce": 3}[args.op], [g])])
    else:
        prog = planner.synthesize(planner.config_path(desc), [n], [0]).placements[0].programs[args.program]
    es = 2 if args.dtype == "bf16" else 4
    elems = (args.mib << 20) // es
    ctx = executor.Context.local(n, list(range(n)), args.mib << 20)
    ctx.set_option("ll_max_bytes", 0)  # one-shot receives wait for peer packets: not profilable alone
    ctx.set_option("push_min_bytes", 0 if args.push else -1)
    if args.reduce_mode is not None:
        ctx.set_option("reduce_mode", args.reduce_mode)
    plan = ctx.compile(prog, elems, args.dtype)
    print("program:", prog.text, "| per-step link bytes per GPU per direction:",
          [plan.step_bytes(s)[0] for s in range(len(prog.steps))], flush=True)
    for _ in range(2):
        plan.run()
    for o in range(n):
        torch.cuda.synchronize(o)
    plan.close()
    ctx.close()


if __name__ == "__main__":
    main()
