"""One process per GPU (the bench's launch shape): CUDA-IPC heaps exchanged
over torch.distributed, each rank enqueues only its own kernels, peers sync
through epoch flags in each other's memory. Compared bit-exactly with the C
oracle on every rank."""
import os

import pytest

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)


def _worker(rank, world, port, result_dir):
    import sys
    import traceback
    import numpy as np
    import torch
    import torch.distributed as dist
    ok = True
    msg = ""
    try:
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
        os.environ["RS_BARRIER_TIMEOUT_S"] = "10"
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from common import golden_programs
        from oracle import numeric
        from paper_2110_10548_b200 import executor
        K = 8
        slot_rank = [d * world // K for d in range(K)]
        ctx = executor.Context.from_process_group(K, slot_rank, 32 << 20)
        for name, N, dt, stride, runs in [("cfg2_r1", 3001, numeric.BF16, 5, 1),
                                          ("cfg2_r01", 4097, numeric.F32, 7, 2),
                                          ("cfg2_r01", 4 << 20, numeric.BF16, 100, 2)]:
            _, progs = golden_programs(name)
            inputs = numeric.synthetic_inputs(K, N, dt)
            es = 2 if dt == numeric.BF16 else 4
            for _, _, prog, _ in progs[::stride]:
                for d in ctx.hosted_slots:
                    ctx.write(d, inputs[d])
                plan = ctx.compile(prog, N, dt)
                for _ in range(runs):
                    plan.run()
                ctx.synchronize()
                want = [x.copy() for x in inputs]
                for _ in range(runs):
                    numeric.execute(prog, K, want, dt)
                for d in ctx.hosted_slots:
                    if not np.array_equal(ctx.read(d, N * es), want[d].view(np.uint8)):
                        raise AssertionError(f"rank {rank} slot {d} mismatch: {prog.text}")
                plan.close()
                dist.barrier()
        # CUDA-graph replay across processes (device-resident epochs)
        _, progs = golden_programs("cfg2_r01")
        N, dt = 2049, numeric.I32
        inputs = numeric.synthetic_inputs(K, N, dt)
        for _, _, prog, _ in progs[::125]:
            plan = ctx.compile(prog, N, dt)
            torch.cuda.synchronize()
            dist.barrier()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                with torch.cuda.graph(g, stream=s):
                    plan.run()
            torch.cuda.synchronize()
            for d in ctx.hosted_slots:
                ctx.write(d, inputs[d])
            torch.cuda.synchronize()
            dist.barrier()
            for _ in range(4):
                g.replay()
            ctx.synchronize()
            want = [x.copy() for x in inputs]
            for _ in range(4):
                numeric.execute(prog, K, want, dt)
            for d in ctx.hosted_slots:
                if not np.array_equal(ctx.read(d, N * 4), want[d].view(np.uint8)):
                    raise AssertionError(f"graph replay mismatch rank {rank} slot {d}: {prog.text}")
            del g
            plan.close()
            dist.barrier()
        dist.barrier()
        ctx.close()
        # One slot per GPU, small buffers: one-shot (LL) steps, eager chains
        # and CUDA-graph replays (packets alternate parity regions by epoch).
        name = {2: "k2_flat", 4: "k4_sock", 8: "k8_sock"}[world]
        K, progs = golden_programs(name)
        ctx = executor.Context.from_process_group(K, list(range(K)), 4 << 20)
        ctx.set_option("ll_total_bytes", 3 << 20)  # one-shot for every size below
        for N, dt in [(1, numeric.BF16), (777, numeric.BF16), (4096, numeric.F32), (30001, numeric.I32)]:
            es = 2 if dt == numeric.BF16 else 4
            inputs = numeric.synthetic_inputs(K, N, dt)
            for _, _, prog, _ in progs[:8]:
                ctx.write(rank, inputs[rank])
                plan = ctx.compile(prog, N, dt)
                if not all(plan.describe()["phase_ll"]):
                    raise AssertionError(f"expected one-shot steps: {prog.text}")
                torch.cuda.synchronize()
                dist.barrier()
                g = torch.cuda.CUDAGraph()
                s = torch.cuda.Stream()
                with torch.cuda.stream(s):
                    plan.run()  # eager run 1
                    with torch.cuda.graph(g, stream=s):
                        plan.run()
                torch.cuda.synchronize()
                for _ in range(6):
                    g.replay()
                ctx.synchronize()
                want = [x.copy() for x in inputs]
                for _ in range(7):
                    numeric.execute(prog, K, want, dt)
                if not np.array_equal(ctx.read(rank, N * es), want[rank].view(np.uint8)):
                    raise AssertionError(f"one-shot replay mismatch rank {rank}: {prog.text} N={N}")
                del g
                plan.close()
                dist.barrier()
        # Push variant across processes: chunk flags live in the owners'
        # heaps (IPC-mapped); eager chains and a graph replay.
        ctx.set_option("push_min_bytes", 0)
        ctx.set_option("ll_max_bytes", 0)
        N, dt = (1 << 20) - 5, numeric.I32
        inputs = numeric.synthetic_inputs(K, N, dt)
        pushed = 0
        for _, _, prog, _ in progs[:6]:
            ctx.write(rank, inputs[rank])
            plan = ctx.compile(prog, N, dt)
            modes = {t["mode"] for st in plan.describe()["steps"] for rk in st["ranks"] for t in rk["tasks"]}
            pushed += 3 in modes  # AllReduce / balanced AllGather steps push
            torch.cuda.synchronize()
            dist.barrier()
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                plan.run()
                plan.run()
                with torch.cuda.graph(g, stream=s):
                    plan.run()
            torch.cuda.synchronize()
            g.replay()
            ctx.synchronize()
            want = [x.copy() for x in inputs]
            for _ in range(3):  # two eager runs + one replay
                numeric.execute(prog, K, want, dt)
            if not np.array_equal(ctx.read(rank, N * 4), want[rank].view(np.uint8)):
                raise AssertionError(f"push mismatch rank {rank}: {prog.text}")
            del g
            plan.close()
            dist.barrier()
        if pushed == 0:
            raise AssertionError("no program used the push variant")
        ctx.close()
        dist.destroy_process_group()
    except Exception:
        ok = False
        msg = traceback.format_exc()
    with open(os.path.join(result_dir, f"r{rank}.txt"), "w") as f:
        f.write("OK" if ok else msg)


@pytest.mark.parametrize("world", [2])
def test_ipc_two_processes(tmp_path, world):
    import socket
    import torch.multiprocessing as mp
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn", join=True)
    for r in range(world):
        text = (tmp_path / f"r{r}.txt").read_text()
        assert text == "OK", text
