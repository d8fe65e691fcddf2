"""Cross-rank kernels on a ONE-GPU box, bit-exact: world = 2, 4 and 8 ranks
emulated on cuda:0 (rs_ctx_create_emulated). Each rank has its own heap —
slot buffers, push scratch, chunk-flag area, one-shot packet area, epoch
inbox — and every launch phase runs all ranks' step kernels as ONE
cooperative launch, so the ranks that spin on each other's flags are
co-resident. The plans are the ones compiled for `world` GPUs: pull over
"peer" pointers, one-shot (LL) packets with parity regions, push landing +
chunk flags (dynamic piece queue, 64 KiB reducing pieces), Reduce by push,
entry/exit epoch barriers, CUDA-graph replays. Each variant is forced
through the C-ABI options and checked (Plan.describe) to have run; results
must equal the C oracle (semantics.cc:259-310 folded as dsl.cc:142-164).

Not marked `multigpu`: this is the driver-visible evidence for the NVLink
code paths on a one-GPU box. (IPC heaps and real NVLink: the multigpu tests,
test_gpu_ranks_processes.py / test_gpu_multiprocess.py.)
"""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

import os  # noqa: E402

from common import golden_programs  # noqa: E402
from oracle import numeric  # noqa: E402
from paper_2110_10548_b200 import executor  # noqa: E402
import ranks_worker  # noqa: E402

os.environ.setdefault("RS_BARRIER_TIMEOUT_S", "20")
ES = {numeric.F32: 4, numeric.BF16: 2, numeric.I32: 4}


def _run_case(ctxs, world, case, used):
    K, progs = golden_programs(case["set"])
    assert K == case["K"]
    if K not in ctxs:
        ctxs[K] = executor.Context.emulated(K, [d * world // K for d in range(K)], world, 0, 8 << 20)
    ctx = ctxs[K]
    for key, value in ranks_worker.VARIANTS[case["variant"]].items():
        ctx.set_option(key, value)
    N, dt = case["N"], case["dtype"]
    inputs = numeric.synthetic_inputs(K, N, dt)
    for _, _, prog, _ in progs[::case["stride"]]:
        for d in range(K):
            ctx.write(d, inputs[d])
        plan = ctx.compile(prog, N, dt)
        desc = plan.describe()
        desc["program_steps"] = prog.steps
        used[case["variant"]] = used.get(case["variant"], 0) + sum(
            ranks_worker._variant_used(case["variant"], desc, r) for r in range(world))
        runs = case["runs"]
        if case.get("graph"):
            g = torch.cuda.CUDAGraph()
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                plan.run()
                with torch.cuda.graph(g, stream=s):
                    plan.run()
            torch.cuda.synchronize()
            for _ in range(runs - 1):
                g.replay()
            del g
        else:
            for _ in range(runs):
                plan.run()
        ctx.synchronize()
        want = [x.copy() for x in inputs]
        for _ in range(runs):
            numeric.execute(prog, K, want, dt)
        for d in range(K):
            got = ctx.read(d, N * ES[dt])
            assert np.array_equal(got, want[d].view(np.uint8)), (
                f"world {world} slot {d}: set={case['set']} variant={case['variant']} N={N} dtype={dt} "
                f"prog={prog.text}")
        plan.close()


@pytest.mark.timeout(1200)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_every_variant(world):
    ctxs, used = {}, {}
    try:
        for case in ranks_worker.default_cases(world):
            _run_case(ctxs, world, case, used)
    finally:
        for c in ctxs.values():
            c.close()
    for variant in ("ll", "pull", "push", "reduce_push"):
        assert used.get(variant, 0) > 0, f"variant {variant} never ran: {used}"


def test_emulated_full_size_push_allreduce():
    """Config-2 size class on the push path at world 4 (16 MiB bf16 per slot,
    many waves of chunk flags through the dynamic piece queue), replayed."""
    world, K = 4, 4
    _, progs = golden_programs("k4_sock")
    ctx = executor.Context.emulated(K, list(range(K)), world, 0, 16 << 20)
    try:
        ctx.set_option("push_min_bytes", 0)
        N = (16 << 20) // 2
        inputs = numeric.synthetic_inputs(K, N, numeric.BF16)
        for _, _, prog, _ in progs[:3]:
            for d in range(K):
                ctx.write(d, inputs[d])
            plan = ctx.compile(prog, N, "bf16")
            for _ in range(3):
                plan.run()
            ctx.synchronize()
            want = [x.copy() for x in inputs]
            for _ in range(3):
                numeric.execute(prog, K, want, numeric.BF16)
            for d in range(K):
                assert np.array_equal(ctx.read(d, N * 2), want[d].view(np.uint8)), (prog.text, d)
            plan.close()
    finally:
        ctx.close()


def _dense_cases(world):
    """Every program of the one-slot-per-rank set and of config 2 (and a
    third of config 3) under each variant."""
    one = ranks_worker.ONE_SLOT_SET[world]
    cases = []
    for variant, N, dt in (("ll", 777, numeric.BF16), ("pull", 4097, numeric.F32),
                           ("push", (1 << 16) + 3, numeric.I32), ("reduce_push", (1 << 16) + 5, numeric.BF16)):
        cases.append({"set": one, "K": world, "N": N, "dtype": dt, "variant": variant, "stride": 1, "runs": 1})
    for name in ("cfg2_r1", "cfg2_r01"):
        cases.append({"set": name, "K": 8, "N": 3001, "dtype": numeric.BF16, "variant": "pull", "stride": 1,
                      "runs": 1})
        cases.append({"set": name, "K": 8, "N": 1001, "dtype": numeric.I32, "variant": "ll", "stride": 1,
                      "runs": 1})
        cases.append({"set": name, "K": 8, "N": (1 << 16) + 3, "dtype": numeric.BF16, "variant": "push",
                      "stride": 3, "runs": 1})
    for name in ("cfg3_r0", "cfg3_r01", "cfg3_r12"):
        cases.append({"set": name, "K": 8, "N": 1001, "dtype": numeric.F32, "variant": "pull", "stride": 3,
                      "runs": 1})
    return cases


@pytest.mark.timeout(1800)
@pytest.mark.parametrize("world", [2, 4, 8])
def test_emulated_ranks_every_program(world):
    ctxs, used = {}, {}
    try:
        for case in _dense_cases(world):
            _run_case(ctxs, world, case, used)
    finally:
        for c in ctxs.values():
            c.close()
    assert all(used.get(v, 0) > 0 for v in ("ll", "pull", "push")), used


@pytest.mark.timeout(1200)
def test_reference_multinode_config_k32_on_one_gpu():
    """The reference's two-node A100 machine (a100_2node.json, axes [8,4],
    reduce {0}: 32 program devices, 254 programs): every program in local mode
    (32 slots on one GPU) and a sample with the 32 slots spread over 8
    emulated ranks (pull and push), bit-exact for bf16 and int32."""
    K, progs = golden_programs("a100_2node_r0")
    assert K == 32
    ctx = executor.Context.local(K, [0] * K, max_bytes=1 << 20)
    try:
        for dt, N in ((numeric.BF16, 2053), (numeric.I32, 1031)):
            inputs = numeric.synthetic_inputs(K, N, dt)
            for _, _, prog, _ in progs:
                for d in range(K):
                    ctx.write(d, inputs[d])
                plan = ctx.compile(prog, N, dt)
                plan.run()
                ctx.synchronize()
                want = [x.copy() for x in inputs]
                numeric.execute(prog, K, want, dt)
                for d in range(K):
                    assert np.array_equal(ctx.read(d, N * ES[dt]), want[d].view(np.uint8)), (prog.text, d)
                plan.close()
    finally:
        ctx.close()
    ctxs, used = {}, {}
    try:
        for variant, N, dt in (("pull", 3001, numeric.BF16), ("push", (1 << 16) + 3, numeric.I32)):
            _run_case(ctxs, 8, {"set": "a100_2node_r0", "K": 32, "N": N, "dtype": dt, "variant": variant,
                                "stride": 9, "runs": 1}, used)
    finally:
        for c in ctxs.values():
            c.close()
    assert used.get("pull", 0) > 0 and used.get("push", 0) > 0, used
