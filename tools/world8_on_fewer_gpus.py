#!/usr/bin/env python
"""Runtime check of the world-8 code paths (8 ranks, IPC among 8 processes,
8-slot barrier sets, 7-peer one-shot and push steps) on a box with fewer
GPUs: rank r drives GPU r % device_count (processes share GPUs, so kernels
time-slice — slow, correctness only). Compares every rank's slot with the C
oracle.
  torchrun --nproc-per-node 8 tools/world8_on_fewer_gpus.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def main():
    os.environ.setdefault("RS_BARRIER_TIMEOUT_S", "20")
    import numpy as np
    import torch
    import torch.distributed as dist
    from common import golden_programs
    from oracle import numeric
    from paper_2110_10548_b200 import executor
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(rank % torch.cuda.device_count())
    dist.init_process_group("gloo", init_method="env://")
    K, progs = golden_programs("k8_sock")
    assert K == world == 8
    ctx = executor.Context.from_process_group(K, list(range(K)), 8 << 20)
    if ctx.nvls:  # RS_NVLS=1: two ranks per GPU cannot share a multicast object -> consistent P2P fallback
        ctx.set_option("nvls_min_bytes", 0)
    bad = 0
    cases = [(4097, numeric.F32, 0, -1), (3001, numeric.BF16, 256 << 10, -1), ((1 << 20) - 3, numeric.I32, 0, 0)]
    for N, dt, ll, push in cases:
        ctx.set_option("ll_max_bytes", ll)
        ctx.set_option("ll_total_bytes", 3 << 20)
        ctx.set_option("push_min_bytes", push)
        es = 2 if dt == numeric.BF16 else 4
        inputs = numeric.synthetic_inputs(K, N, dt)
        for _, _, prog, _ in progs[:3]:
            ctx.write(rank, inputs[rank])
            plan = ctx.compile(prog, N, dt)
            plan.run()
            ctx.synchronize()
            want = [x.copy() for x in inputs]
            numeric.execute(prog, K, want, dt)
            ok = np.array_equal(ctx.read(rank, N * es), want[rank].view(np.uint8))
            bad += 0 if ok else 1
            plan.close()
            dist.barrier()
    t = torch.tensor([bad])
    dist.all_reduce(t)
    if rank == 0:
        print(f"world {world} on {torch.cuda.device_count()} GPUs (RS_NVLS={os.environ.get('RS_NVLS', '0')}, "
              f"nvls after compiles: {ctx.nvls}): mismatches={int(t.item())}", flush=True)
    ctx.close()
    dist.destroy_process_group()
    return 0 if int(t.item()) == 0 else 1


if __name__ == "__main__":
    sys.exit(main())
