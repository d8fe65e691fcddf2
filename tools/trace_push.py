#!/usr/bin/env python
"""Piece timeline of one cross-GPU step (profiling build only): every CTA's
thread 0 stamps %globaltimer at each piece's start, "inputs ready" (after the
chunk-flag waits of a push reducing piece / before the flag store of a landing
piece) and end, plus each CTA's entry and entry-barrier exit. One process per
GPU; writes the raw stamps of every rank to --out (JSON) and prints a summary.

  make profiling
  torchrun --nproc-per-node 4 tools/trace_push.py --op reduce --mib 1024 --reduce-mode 1 --wave-mib 16
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

OPS = {"allreduce": 0, "reducescatter": 1, "allgather": 2, "reduce": 3, "broadcast": 4}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--op", default="allreduce", choices=list(OPS))
    ap.add_argument("--mib", type=int, default=64)
    ap.add_argument("--reduce-mode", type=int, default=0)
    ap.add_argument("--wave-mib", type=int, default=0)
    ap.add_argument("--push-min-mib", type=int, default=32, help="-1: never push")
    ap.add_argument("--runs", type=int, default=4)
    ap.add_argument("--out", default=None)
    args = ap.parse_args()
    prof = os.path.join(ROOT, "paper_2110_10548_b200", "_lib", "libredsynth_b200_prof.so")
    if not os.path.exists(prof):
        raise SystemExit("build the profiling library first: make profiling")
    os.environ["RS_LIB_PATH"] = prof
    import torch
    import torch.distributed as dist
    from paper_2110_10548_b200 import executor
    from paper_2110_10548_b200.planner import LoweredProgram
    world, rank = int(os.environ["WORLD_SIZE"]), int(os.environ["RANK"])
    torch.cuda.set_device(rank)
    dev = torch.device("cuda", rank)
    dist.init_process_group("gloo")
    ctx = executor.Context.from_process_group(world, list(range(world)), args.mib << 20)
    ctx.set_option("ll_max_bytes", 0)
    ctx.set_option("push_min_bytes", -1 if args.push_min_mib < 0 else args.push_min_mib << 20)
    ctx.set_option("reduce_mode", args.reduce_mode)
    ctx.set_option("push_wave_bytes", args.wave_mib << 20)
    prog = LoweredProgram(steps=[(OPS[args.op], [list(range(world))])])
    elems = (args.mib << 20) // 2
    gen = torch.Generator(device=dev)
    gen.manual_seed(1000 + rank)
    ctx.buffer(rank, elems, "bf16").copy_(torch.randn(elems, generator=gen, device=dev).to(torch.bfloat16))
    plan = ctx.compile(prog, elems, "bf16")
    desc = plan.describe()
    me = desc["steps"][0]["ranks"][rank]
    npieces = me["npieces"]
    trace = torch.zeros(3 * npieces + 2 * 4096, dtype=torch.int64, device=dev)
    os.environ["RS_TRACE_PTR"] = str(trace.data_ptr())
    torch.cuda.synchronize()
    dist.barrier()
    for _ in range(args.runs):
        plan.run()
    ctx.synchronize()
    t = trace.cpu().tolist()
    modes = []
    for i, task in enumerate(me["tasks"]):
        last = me["tasks"][i + 1]["piece_begin"] if i + 1 < len(me["tasks"]) else npieces
        modes += [task["mode"]] * (last - task["piece_begin"])
    pieces = [(modes[p], t[3 * p], t[3 * p + 1], t[3 * p + 2]) for p in range(npieces)]
    ctas = [(t[3 * npieces + 2 * b], t[3 * npieces + 2 * b + 1]) for b in range(4096) if t[3 * npieces + 2 * b]]
    rec = {"rank": rank, "pieces": pieces, "ctas": ctas, "tx": me["tx"], "rx": me["rx"]}
    allrec = [None] * world
    dist.all_gather_object(allrec, rec)
    if rank == 0:
        t0 = min(min(c[0] for c in r["ctas"]) for r in allrec)
        print(f"{args.op} {args.mib} MiB bf16, K={world}, reduce_mode={args.reduce_mode}, wave={args.wave_mib} MiB "
              f"(times in us from the earliest CTA entry over all GPUs)")
        for r in allrec:
            ent = [c[0] - t0 for c in r["ctas"]]
            bar = [c[1] - t0 for c in r["ctas"]]
            line = [f"rank {r['rank']}: ctas {len(ent)} entry {min(ent) / 1e3:.1f}-{max(ent) / 1e3:.1f} "
                    f"barrier {min(bar) / 1e3:.1f}-{max(bar) / 1e3:.1f}"]
            for m in sorted({p[0] for p in r["pieces"]}):
                ps = [p for p in r["pieces"] if p[0] == m and p[3]]
                if not ps:
                    continue
                st = sorted(p[1] - t0 for p in ps)
                en = sorted(p[3] - t0 for p in ps)
                wait = sorted(p[2] - p[1] for p in ps) if m == 4 else None
                q = lambda v, f: v[min(len(v) - 1, int(f * len(v)))] / 1e3
                s = (f"mode {m}: {len(ps)} pieces start {q(st, 0):.1f}..{q(st, 1):.1f} end p10 {q(en, .1):.1f} "
                     f"p50 {q(en, .5):.1f} p90 {q(en, .9):.1f} max {q(en, 1):.1f}")
                if wait:
                    s += f" flag-wait p50 {q(wait, .5):.1f} p90 {q(wait, .9):.1f} max {q(wait, 1):.1f}"
                line.append(s)
            line.append(f"tx {r['tx'] / 2**20:.0f} MiB rx {r['rx'] / 2**20:.0f} MiB")
            print("\n  ".join(line), flush=True)
        if args.out:
            with open(args.out, "w") as f:
                json.dump({"args": vars(args), "t0": t0, "ranks": allrec}, f)
    dist.barrier()
    plan.close()
    ctx.close()
    dist.destroy_process_group()


if __name__ == "__main__":
    main()
