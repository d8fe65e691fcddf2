"""Worker of the multi-rank parity tests (one process per rank, the bench's
launch shape): CUDA-IPC heaps exchanged over a gloo process group, each rank
enqueues only its own kernels and synchronises with its peers through epoch
flags in their memory. Compared bit-exactly with the C oracle on every rank.

Rank r runs on cuda:r (test_gpu_ranks_processes.py, multi-GPU boxes).
Ranks must not share a GPU: kernels that spin on each other's flags are not
guaranteed to be co-scheduled as separate launches (and have raised Xid 109
on B200); one-GPU boxes use emulated ranks in one cooperative launch instead.

Each case forces one variant through the context options the C-ABI exposes
(ll_max_bytes, push_min_bytes) and checks from Plan.describe() that the
variant really ran. Anchor: /root/reference/proj/src/semantics.cc:259-310
folded as dsl.cc:142-164 (oracle/numeric.c).
"""
import json
import os
import sys
import traceback

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)

MODE_SUM, MODE_NVLS, MODE_LL, MODE_FLAG_SEND, MODE_FLAG_RECV = 0, 1, 2, 3, 4
VARIANTS = {
    # name: context options
    "ll": {"ll_max_bytes": 256 << 10, "ll_total_bytes": 3 << 20, "push_min_bytes": -1, "reduce_mode": 0},
    "pull": {"ll_max_bytes": 0, "push_min_bytes": -1, "reduce_mode": 0},
    "push": {"ll_max_bytes": 0, "push_min_bytes": 0, "reduce_mode": 0},
    # Reduce over >= 3 ranks by push (stores only, chunk flags) — the other
    # ops as in "push"
    "reduce_push": {"ll_max_bytes": 0, "push_min_bytes": 0, "reduce_mode": 1},
}
ONE_SLOT_SET = {2: "k2_flat", 4: "k4_sock", 8: "k8_sock"}


def _modes(desc, rank):
    """Task modes rank `rank` executes, and whether any of its pull tasks
    reads or writes another rank's slot."""
    slot_rank = desc["slot_rank"]
    modes, remote_pull = set(), False
    for st in desc["steps"]:
        for t in st["ranks"][rank]["tasks"]:
            modes.add(t["mode"])
            if t["mode"] == MODE_SUM:
                remote_pull |= any(slot_rank[s] != rank for s in t["src"] + t["dst"])
    return modes, remote_pull


def _variant_used(name, desc, rank):
    modes, remote_pull = _modes(desc, rank)
    if name == "ll":
        return all(desc["phase_ll"])
    if name == "push":
        return MODE_FLAG_SEND in modes or MODE_FLAG_RECV in modes
    if name == "reduce_push":
        for st, (op, groups) in zip(desc["steps"], desc["program_steps"]):
            if op != 3 or max(len(g) for g in groups) < 3:
                continue
            if any(t["mode"] in (MODE_FLAG_SEND, MODE_FLAG_RECV) for t in st["ranks"][rank]["tasks"]):
                return True
        return False
    return remote_pull and not (modes & {MODE_LL, MODE_FLAG_SEND, MODE_FLAG_RECV})


def worker(rank, world, port, result_dir, device_of_rank, cases):
    """cases: list of dicts {set, K, N, dtype, variant, stride, runs, graph}."""
    ok, msg, used = True, "", {}
    try:
        sys.path.insert(0, ROOT)
        sys.path.insert(0, HERE)
        os.environ.setdefault("RS_BARRIER_TIMEOUT_S", "60")
        import numpy as np
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(device_of_rank(rank))
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from common import golden_programs
        from oracle import numeric
        from paper_2110_10548_b200 import executor
        ctxs = {}

        def context(K):
            if K not in ctxs:
                slot_rank = [d * world // K for d in range(K)]
                ctxs[K] = executor.Context.from_process_group(K, slot_rank, 8 << 20)
            return ctxs[K]

        for case in cases:
            K, progs = golden_programs(case["set"])
            assert K == case["K"], (K, case)
            ctx = context(K)
            for key, value in VARIANTS[case["variant"]].items():
                ctx.set_option(key, value)
            N, dt = case["N"], case["dtype"]
            es = 2 if dt == numeric.BF16 else 4
            inputs = numeric.synthetic_inputs(K, N, dt)
            for _, _, prog, _ in progs[::case["stride"]]:
                for d in ctx.hosted_slots:
                    ctx.write(d, inputs[d])
                plan = ctx.compile(prog, N, dt)
                desc = plan.describe()
                desc["program_steps"] = prog.steps
                key = f"{case['variant']}"
                used[key] = used.get(key, 0) + (1 if _variant_used(case["variant"], desc, rank) else 0)
                torch.cuda.synchronize()
                dist.barrier()
                runs = case["runs"]
                if case.get("graph"):
                    # eager run, then a captured run replayed (device-resident
                    # epochs; one-shot packets alternate parity regions)
                    g = torch.cuda.CUDAGraph()
                    s = torch.cuda.Stream()
                    with torch.cuda.stream(s):
                        plan.run()
                        with torch.cuda.graph(g, stream=s):
                            plan.run()
                    torch.cuda.synchronize()
                    for _ in range(runs - 1):
                        g.replay()
                    torch.cuda.synchronize()
                    del g
                else:
                    for _ in range(runs):
                        plan.run()
                ctx.synchronize()
                want = [x.copy() for x in inputs]
                for _ in range(runs):
                    numeric.execute(prog, K, want, dt)
                for d in ctx.hosted_slots:
                    if not np.array_equal(ctx.read(d, N * es), want[d].view(np.uint8)):
                        raise AssertionError(f"rank {rank} slot {d} mismatch: set={case['set']} "
                                             f"variant={case['variant']} N={N} dtype={dt} prog={prog.text}")
                plan.close()
                dist.barrier()
        dist.barrier()
        for c in ctxs.values():
            c.close()
        dist.destroy_process_group()
    except Exception:
        ok = False
        msg = traceback.format_exc()
    with open(os.path.join(result_dir, f"r{rank}.json"), "w") as f:
        json.dump({"ok": ok, "msg": msg, "used": used}, f)


def default_cases(world):
    """Every variant x dtype on the one-slot-per-rank golden set (ragged
    sizes, graph replays), plus config-2 / config-3 samples with the 8 slots
    block-distributed over the ranks."""
    from oracle import numeric
    one = ONE_SLOT_SET[world]
    cases = []
    for variant in ("ll", "pull", "push"):
        sizes = [(1, numeric.BF16), (777, numeric.BF16), (4097, numeric.F32), (30001, numeric.I32)]
        if variant != "ll":
            sizes.append(((1 << 18) - 3, numeric.BF16))
        for N, dt in sizes:
            cases.append({"set": one, "K": world, "N": N, "dtype": dt, "variant": variant,
                          "stride": {2: 1, 4: 5, 8: 25}[world], "runs": 2, "graph": N % 2 == 1})
    for N, dt in [(4097, numeric.F32), ((1 << 17) + 5, numeric.BF16), (30001, numeric.I32)]:
        cases.append({"set": one if world > 2 else "k4_sock", "K": max(world, 4), "N": N, "dtype": dt,
                      "variant": "reduce_push", "stride": 7, "runs": 2, "graph": dt == numeric.BF16})
    if world in (2, 4):
        for variant in ("ll", "pull", "push"):
            cases.append({"set": "cfg2_r01", "K": 8, "N": 3001, "dtype": numeric.BF16, "variant": variant,
                          "stride": 50, "runs": 2, "graph": variant == "push"})
            cases.append({"set": "cfg3_r01", "K": 8, "N": 1001, "dtype": numeric.F32, "variant": variant,
                          "stride": 125, "runs": 1, "graph": False})
            cases.append({"set": "cfg2_r1", "K": 8, "N": (1 << 16) + 3, "dtype": numeric.I32, "variant": variant,
                          "stride": 60, "runs": 2, "graph": variant == "ll"})
    return cases


def spawn(world, tmp_path, device_of_rank, cases=None):
    """Runs the worker on `world` processes; returns the per-rank results."""
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    if cases is None:
        cases = default_cases(world)
    mp.start_processes(worker, args=(world, port, str(tmp_path), device_of_rank, cases), nprocs=world,
                       start_method="spawn", join=True)
    out = []
    for r in range(world):
        with open(os.path.join(str(tmp_path), f"r{r}.json")) as f:
            out.append(json.load(f))
    return out


def on_own_gpu(rank):
    return rank
