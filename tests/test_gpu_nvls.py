"""NVLS (multimem.ld_reduce / multimem.st through the NVSwitch) variant.

The switch sums in its own order, so f32/bf16 results are checked against the
exact group sum within the stated bound
    |y - sum_j x_j| <= S * (n * 2^-24 + r) * sum_j |x_j|,   r = n 2^-8 (bf16) or 0 (f32)
(measured on B200: the switch's bf16 ld_reduce is not correctly rounded even
with .acc::f32 — ~1.5 ulp on ~2% of elements at n = 4, and at n = 2 results
off by up to ~0.75 ulp on 19% of elements, profiles/r01_nvls_bf16_n2_rounding.txt)
(S = program steps, n = reduction-group size), and every member of a
reduction group must hold bit-identical results. int32 never uses NVLS and
stays bit-exact.
"""
import os

import numpy as np
import pytest

from common import bf16_widen, golden_programs
from oracle import numeric

pytestmark = [pytest.mark.gpu, pytest.mark.multigpu]

torch = pytest.importorskip("torch")
if not torch.cuda.is_available() or torch.cuda.device_count() < 2:
    pytest.skip("needs >= 2 GPUs", allow_module_level=True)

from paper_2110_10548_b200 import executor  # noqa: E402

NGPU = torch.cuda.device_count()
ES = {numeric.F32: 4, numeric.BF16: 2, numeric.I32: 4}


def _as_f64(raw, dtype):
    if dtype == numeric.F32:
        return raw.view(np.float32).astype(np.float64)
    if dtype == numeric.BF16:
        return bf16_widen(raw.view(np.uint16)).astype(np.float64)
    return raw.view(np.int32).astype(np.int64)


def check_within_bound(prog, part, inputs, outputs, dtype):
    S = max(1, len(prog.steps))
    for grp in part:
        n = len(grp)
        xs = [_as_f64(inputs[d].view(np.uint8), dtype) for d in grp]
        exact = np.sum(xs, axis=0)
        mag = np.sum(np.abs(xs), axis=0)
        # the switch's bf16 sums are not correctly rounded (see module doc)
        r = n * 2.0 ** -8 if dtype == numeric.BF16 else 0.0
        tol = S * (n * 2.0 ** -24 + r) * mag + 1e-30
        first = outputs[grp[0]]
        for d in grp:
            assert np.array_equal(outputs[d], first), (prog.text, "replicas differ", d)
            y = _as_f64(outputs[d], dtype)
            if dtype == numeric.I32:
                assert np.array_equal(y, exact.astype(np.int32).astype(np.int64))
            else:
                bad = np.abs(y - exact) > tol
                assert not bad.any(), (prog.text, d, int(bad.sum()), float(np.max(np.abs(y - exact) - tol)))


def _run(ctx, prog, part, K, N, dtype, runs=1):
    inputs = numeric.synthetic_inputs(K, N, dtype)
    for d in range(K):
        ctx.write(d, inputs[d])
    plan = ctx.compile(prog, N, dtype)
    d0 = plan.describe()
    nvls_tasks = sum(1 for st in d0["steps"] for rk in st["ranks"] for t in rk["tasks"] if t.get("mode") == 1)
    plan.run()
    ctx.synchronize()
    outs = [ctx.read(d, N * ES[dtype]) for d in range(K)]
    check_within_bound(prog, part, inputs, outs, dtype)
    plan.close()
    return nvls_tasks


@pytest.fixture(scope="module")
def nvls_ctx():
    n = 4 if NGPU >= 4 else 2
    os.environ["RS_NVLS"] = "1"
    try:
        ctx = executor.Context.local(n, list(range(n)), max_bytes=64 << 20)
    finally:
        os.environ.pop("RS_NVLS", None)
    if not ctx.nvls:
        ctx.close()
        pytest.skip("multicast not supported")
    if n == 2:
        ctx.set_option("nvls_min_group", 2)
    ctx.set_option("nvls_min_bytes", 0)  # exercise NVLS at every size
    ctx.set_option("ll_max_bytes", 0)  # (one-shot would take the small ones)
    yield ctx, n
    ctx.close()


@pytest.mark.parametrize("dtype", [numeric.F32, numeric.BF16])
def test_nvls_programs_within_bound(nvls_ctx, dtype):
    ctx, n = nvls_ctx
    name = {2: "k2_flat", 4: "k4_sock"}[n]
    K, progs = golden_programs(name)
    used = 0
    for _, _, prog, part in progs:
        for N in (4099, 1 << 20):
            used += _run(ctx, prog, part, K, N, dtype)
    assert used > 0, "no program used NVLS"


def test_nvls_int32_stays_exact(nvls_ctx):
    ctx, n = nvls_ctx
    name = {2: "k2_flat", 4: "k4_sock"}[n]
    K, progs = golden_programs(name)
    for _, _, prog, part in progs[:20]:
        assert _run(ctx, prog, part, K, 3001, numeric.I32) == 0


def test_nvls_large_allreduce_repeated(nvls_ctx):
    ctx, n = nvls_ctx
    name = {2: "k2_flat", 4: "k4_flat"}[n]
    K, progs = golden_programs(name)
    prog, part = progs[0][2], progs[0][3]
    N = 16 << 20
    inputs = numeric.synthetic_inputs(K, N, numeric.BF16)
    for d in range(K):
        ctx.write(d, inputs[d])
    plan = ctx.compile(prog, N, "bf16")
    for _ in range(3):  # in place: inputs grow by n per run; check the first run only below
        pass
    plan.run()
    ctx.synchronize()
    outs = [ctx.read(d, N * 2) for d in range(K)]
    check_within_bound(prog, part, inputs, outs, numeric.BF16)
    for _ in range(5):
        plan.run()
    ctx.synchronize()
    plan.close()


def _mp_worker(rank, world, port, result_dir):
    import sys
    import traceback
    ok, msg = True, ""
    try:
        here = os.path.dirname(os.path.abspath(__file__))
        sys.path.insert(0, os.path.dirname(here))
        sys.path.insert(0, here)
        os.environ["RS_NVLS"] = "1"
        os.environ["RS_BARRIER_TIMEOUT_S"] = "10"
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(rank)
        dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
        from common import golden_programs
        from oracle import numeric
        from paper_2110_10548_b200 import executor
        from test_gpu_nvls import check_within_bound
        name = {2: "k2_flat", 4: "k4_sock"}[world]
        K, progs = golden_programs(name)
        ctx = executor.Context.from_process_group(K, list(range(K)), 32 << 20)
        assert ctx.nvls, "NVLS not enabled"
        if world == 2:
            ctx.set_option("nvls_min_group", 2)
        ctx.set_option("nvls_min_bytes", 0)
        ctx.set_option("ll_max_bytes", 0)
        used = 0
        for dt in (numeric.BF16, numeric.F32):
            for N in (5003, 4 << 20):
                inputs = numeric.synthetic_inputs(K, N, dt)
                for _, _, prog, part in progs[::3]:
                    ctx.write(rank, inputs[rank])
                    plan = ctx.compile(prog, N, dt)
                    used += sum(1 for st in plan.describe()["steps"] for rk in st["ranks"]
                                for t in rk["tasks"] if t.get("mode") == 1)
                    plan.run()
                    ctx.synchronize()
                    mine = ctx.read(rank, N * (2 if dt == numeric.BF16 else 4))
                    gathered = [None] * world
                    dist.all_gather_object(gathered, mine.tobytes())
                    outs = [np.frombuffer(b, dtype=np.uint8) for b in gathered]
                    check_within_bound(prog, part, inputs, outs, dt)
                    plan.close()
                    dist.barrier()
        assert used > 0
        dist.barrier()
        ctx.close()
        dist.destroy_process_group()
    except Exception:
        ok, msg = False, traceback.format_exc()
    with open(os.path.join(result_dir, f"r{rank}.txt"), "w") as f:
        f.write("OK" if ok else msg)


def test_nvls_one_process_per_gpu(tmp_path):
    """Multi-process NVLS: heaps shared as fds (pidfd_getfd), multicast
    objects created collectively through the host exchange callback."""
    import socket
    import torch.multiprocessing as mp
    world = 4 if NGPU >= 4 else 2
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    mp.start_processes(_mp_worker, args=(world, port, str(tmp_path)), nprocs=world, start_method="spawn", join=True)
    for r in range(world):
        text = (tmp_path / f"r{r}.txt").read_text()
        assert text == "OK", text


def test_nvls_broadcast_bit_exact(nvls_ctx):
    """NVLS Broadcast (the root's bytes stored once to the multicast address,
    the switch writes every member) is a bit copy: programs whose only
    multicast steps are Broadcasts stay bit-exact for every dtype, and the
    Broadcast steps really use multicast tasks (mode 6)."""
    from paper_2110_10548_b200.planner import LoweredProgram
    ctx, n = nvls_ctx
    g = list(range(n))
    prog = LoweredProgram(steps=[(3, [g]), (4, [g])])  # Reduce then Broadcast
    for dtype in (numeric.I32, numeric.BF16, numeric.F32):
        for N in (4099, (8 << 20) + 5):
            ctx.set_option("reduce_mode", 0)  # exact P2P Reduce; NVLS only in the Broadcast
            ctx.set_option("nvls_bcast", 1)
            inputs = numeric.synthetic_inputs(n, N, dtype)
            for d in range(n):
                ctx.write(d, inputs[d])
            plan = ctx.compile(prog, N, dtype)
            desc = plan.describe()
            modes = {t["mode"] for rk in desc["steps"][1]["ranks"] for t in rk["tasks"]}
            assert 6 in modes, modes
            for _ in range(2):
                plan.run()
            ctx.synchronize()
            want = [x.copy() for x in inputs]
            for _ in range(2):
                numeric.execute(prog, n, want, dtype)
            for d in range(n):
                assert np.array_equal(ctx.read(d, N * ES[dtype]), want[d].view(np.uint8)), (dtype, N, d)
            plan.close()
    ctx.set_option("reduce_mode", -1)
    ctx.set_option("nvls_bcast", 0)
