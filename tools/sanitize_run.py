#!/usr/bin/env python
"""Small executor workload for compute-sanitizer (memcheck / racecheck /
synccheck): local mode (8 slots on cuda:0, every collective as HBM-local
tasks) and, with --world 2, two processes on cuda:0 and cuda:1 joined by CUDA
IPC (the cross-rank pull, one-shot and push kernels with their flag
protocol). (compute-sanitizer was closed on this round's GPU pool.)
Bit-exact against the C oracle; exits non-zero on a mismatch.
  compute-sanitizer --tool memcheck --target-processes all python tools/sanitize_run.py --world 2"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def local():
    import numpy as np
    from common import golden_programs
    from oracle import numeric
    from paper_2110_10548_b200 import executor
    ctx = executor.Context.local(8, [0] * 8, 1 << 20)
    K, progs = golden_programs("cfg2_r01")
    bad = 0
    for dt, N in ((numeric.BF16, 4097), (numeric.F32, 1001), (numeric.I32, 333)):
        es = 2 if dt == numeric.BF16 else 4
        inputs = numeric.synthetic_inputs(K, N, dt)
        for _, _, prog, _ in progs[::50]:
            for d in range(K):
                ctx.write(d, inputs[d])
            plan = ctx.compile(prog, N, dt)
            plan.run()
            ctx.synchronize()
            want = [x.copy() for x in inputs]
            numeric.execute(prog, K, want, dt)
            bad += sum(not np.array_equal(ctx.read(d, N * es), want[d].view(np.uint8)) for d in range(K))
            plan.close()
    ctx.close()
    print(f"local: mismatches={bad}", flush=True)
    return bad


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--world", type=int, default=1)
    args = ap.parse_args()
    os.environ.setdefault("RS_BARRIER_TIMEOUT_S", "300")
    if args.world == 1:
        return 1 if local() else 0
    import tempfile
    import ranks_worker
    from oracle import numeric
    cases = []
    for variant in ("ll", "pull", "push", "reduce_push"):
        cases.append({"set": "k4_sock", "K": 4, "N": 3001 if variant == "ll" else (1 << 16) + 3,
                      "dtype": numeric.BF16, "variant": variant, "stride": 40, "runs": 2, "graph": False})
    with tempfile.TemporaryDirectory() as tmp:
        res = ranks_worker.spawn(args.world, tmp, ranks_worker.on_own_gpu, cases)
    ok = all(r["ok"] for r in res)
    print(f"world {args.world}: {'OK' if ok else 'FAILED'} used={res[0]['used']}", flush=True)
    if not ok:
        for r in res:
            print(r["msg"])
    return 0 if ok else 1


if __name__ == "__main__":
    sys.exit(main())
