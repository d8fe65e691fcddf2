"""GPU parity: the sm_100a executor against the C oracle, through the C-ABI.

Bit-exact for every dtype (the kernels sum members in the oracle's order and
round bf16 once), on every synthesized program of configs 1-3, plus full-size
BASELINE buffers, several slot->GPU mappings, repeated runs (epoch flags),
the user-buffer and host-buffer paths and refusal behaviour.
"""
import os

import numpy as np
import pytest

from common import golden_programs
from oracle import numeric

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

from paper_2110_10548_b200 import executor  # noqa: E402
from paper_2110_10548_b200._native import ExecError  # noqa: E402

os.environ.setdefault("RS_BARRIER_TIMEOUT_S", "10")
ES = {numeric.F32: 4, numeric.BF16: 2, numeric.I32: 4}
NGPU = torch.cuda.device_count()


def _run(ctx, prog, K, N, dtype, inputs=None, runs=1):
    inputs = inputs if inputs is not None else numeric.synthetic_inputs(K, N, dtype)
    for d in range(K):
        ctx.write(d, inputs[d])
    plan = ctx.compile(prog, N, dtype)
    for _ in range(runs):
        plan.run()
    ctx.synchronize()
    got = [ctx.read(d, N * ES[dtype]) for d in range(K)]
    want = [x.copy() for x in inputs]
    for _ in range(runs):
        numeric.execute(prog, K, want, dtype)
    for d in range(K):
        assert np.array_equal(got[d], want[d].view(np.uint8)), (prog.text, d)
    plan.close()


@pytest.fixture(scope="module")
def local8():
    ctx = executor.Context.local(8, [0] * 8, max_bytes=256 << 20)
    yield ctx
    ctx.close()


@pytest.mark.parametrize("dtype", [numeric.F32, numeric.BF16, numeric.I32])
def test_config1_every_program_local(local8, dtype):
    K, progs = golden_programs("cfg1")
    for _, _, prog, _ in progs:
        _run(local8, prog, K, 4099, dtype)


def test_config1_full_size_f32_local(local8):
    """Config 1 exactly: 64 MiB fp32 per device, all 8 synthesized programs."""
    K, progs = golden_programs("cfg1")
    N = 16 * 1024 * 1024
    inputs = numeric.synthetic_inputs(K, N, numeric.F32)
    for _, _, prog, _ in progs:
        _run(local8, prog, K, N, numeric.F32, inputs=inputs)


@pytest.mark.parametrize("name", ["cfg2_r1", "cfg2_r01"])
def test_config2_every_program_bf16_local(local8, name):
    K, progs = golden_programs(name)
    for _, _, prog, _ in progs:
        _run(local8, prog, K, 2053, numeric.BF16)


def test_config2_full_size_bf16_local(local8):
    """256 MiB bf16 per device (config 2's size) on a sample of programs."""
    K, progs = golden_programs("cfg2_r01")
    N = 128 * 1024 * 1024
    inputs = numeric.synthetic_inputs(K, N, numeric.BF16)
    for _, _, prog, _ in progs[::125]:
        _run(local8, prog, K, N, numeric.BF16, inputs=inputs)


@pytest.mark.parametrize("queue", [-1, 0, 1, 2])
def test_piece_schedules_local(local8, queue):
    """Static grid stride (piece_queue 0) and the prefetched atomic queue
    (-1 auto, 1, 2): the same bytes, bit-exact, replayed (the queue word resets at
    the end of each launch). describe() after a run reports the schedule:
    the queue only on phases with >= 2 pieces per CTA."""
    K, progs = golden_programs("cfg2_r01")
    for N in (12 << 20, 100003):
        inputs = numeric.synthetic_inputs(K, N, numeric.BF16)
        for _, _, prog, _ in progs[::125]:
            for d in range(K):
                local8.write(d, inputs[d])
            plan = local8.compile(prog, N, numeric.BF16)
            plan.set_option("piece_queue", queue)
            for _ in range(3):
                plan.run()
            local8.synchronize()
            want = [x.copy() for x in inputs]
            for _ in range(3):
                numeric.execute(prog, K, want, numeric.BF16)
            for d in range(K):
                assert np.array_equal(local8.read(d, N * 2), want[d].view(np.uint8)), (prog.text, queue, N, d)
            for st in plan.describe()["steps"]:
                rk = st["ranks"][0]
                expect = 2 if queue and rk["npieces"] >= 2 * rk["grid"] else 0
                assert rk["queue"] == expect, (prog.text, queue, N, rk["npieces"], rk["grid"], rk["queue"])
            plan.close()


@pytest.mark.parametrize("name", ["cfg3_r0", "cfg3_r1", "cfg3_r2", "cfg3_r01", "cfg3_r02", "cfg3_r12"])
def test_config3_every_program_f32_local(local8, name):
    K, progs = golden_programs(name)
    for _, _, prog, _ in progs:
        _run(local8, prog, K, 1001, numeric.F32)


@pytest.mark.parametrize("N", [0, 1, 7, 8, 9, 33, 1023, 65537])
def test_ragged_sizes_local(local8, N):
    K, progs = golden_programs("cfg2_r01")
    for _, _, prog, _ in progs[::40]:
        for dt in (numeric.BF16, numeric.I32):
            _run(local8, prog, K, N, dt)


def test_repeated_runs_chain(local8):
    K, progs = golden_programs("cfg2_r1")
    for _, _, prog, _ in progs[::50]:
        _run(local8, prog, K, 5000, numeric.I32, runs=3)


def test_cuda_graph_replay(local8):
    """plan.run() captured in a CUDA graph and replayed: epochs are device
    resident, so replays chain exactly like eager runs."""
    K, progs = golden_programs("cfg2_r01")
    N = 3001
    for _, _, prog, _ in progs[::100]:
        inputs = numeric.synthetic_inputs(K, N, numeric.I32)
        for d in range(K):
            local8.write(d, inputs[d])
        plan = local8.compile(prog, N, "i32")
        torch.cuda.synchronize()
        g = torch.cuda.CUDAGraph()
        s = torch.cuda.Stream()
        with torch.cuda.stream(s):
            plan.run()  # warm-up outside capture (state advances: counts as run 1)
            with torch.cuda.graph(g, stream=s):
                plan.run()
        torch.cuda.synchronize()
        for d in range(K):
            local8.write(d, inputs[d])
        for _ in range(3):
            g.replay()
        local8.synchronize()
        want = [x.copy() for x in inputs]
        for _ in range(3):
            numeric.execute(prog, K, want, numeric.I32)
        for d in range(K):
            assert np.array_equal(local8.read(d, N * 4), want[d].view(np.uint8))
        del g
        plan.close()


def test_user_and_host_buffer_paths(local8):
    K, progs = golden_programs("cfg2_r01")
    N = 10007
    prog = progs[123][2]
    inputs = numeric.synthetic_inputs(K, N, numeric.F32)
    want = [x.copy() for x in inputs]
    numeric.execute(prog, K, want, numeric.F32)
    plan = local8.compile(prog, N, "f32")
    dev = [torch.from_numpy(x.copy()).cuda() for x in inputs]
    plan.run(bufs=dev)
    local8.synchronize()
    for d in range(K):
        assert np.array_equal(dev[d].cpu().numpy(), want[d])
    host = [torch.from_numpy(x.copy()).pin_memory() for x in inputs]
    plan.run_host(host)
    local8.synchronize()
    for d in range(K):
        assert np.array_equal(host[d].numpy(), want[d])


def test_upload_run_download_stream_ordered(local8):
    """rs_ctx_upload -> several plans in place -> rs_ctx_download, all async on
    torch's current stream: results equal the oracle applied in sequence."""
    K, progs = golden_programs("cfg2_r01")
    N = 1 << 20
    inputs = numeric.synthetic_inputs(K, N, numeric.I32)
    host_in = [torch.from_numpy(x.copy()).pin_memory() for x in inputs]
    host_out = [torch.empty_like(t).pin_memory() for t in host_in]
    chain = [progs[i][2] for i in (0, 77, 311)]
    plans = [local8.compile(p, N, "i32") for p in chain]
    for d in range(K):
        local8.upload(d, host_in[d])
    for p in plans:
        p.run()
    for d in range(K):
        local8.download(d, host_out[d])
    torch.cuda.current_stream().synchronize()
    want = [x.copy() for x in inputs]
    for p in chain:
        numeric.execute(p, K, want, numeric.I32)
    for d in range(K):
        assert np.array_equal(host_out[d].numpy(), want[d])
    for p in plans:
        p.close()


def test_refusal_launches_nothing(local8):
    from paper_2110_10548_b200.planner import LoweredProgram
    bad = LoweredProgram(steps=[(3, [[0, 1, 2, 3]]), (3, [[0, 1, 2, 3]])])
    with pytest.raises(ExecError) as e:
        local8.compile(bad, 100, "f32")
    assert e.value.code == 9
    assert e.value.message == "step 1: Reduce over devices {0,1,2,3}: devices hold different chunk sets"
    K, progs = golden_programs("cfg1")  # the context still works afterwards
    _run(local8, progs[0][2], K, 100, numeric.F32)


def test_plan_time_and_prediction(local8):
    """rs_plan_time (device time of a run) and the calibrated prediction
    agree within a factor of two on a full-size config-2 program."""
    K, progs = golden_programs("cfg2_r01")
    plan = local8.compile(progs[0][2], 128 * 1024 * 1024, "bf16")
    us = plan.time_us(1, 3)
    pred = plan.predict_us(3.0, 650.0, 5967.0)
    assert us > 0 and 0.5 < us / pred < 2.0, (us, pred)
    plan.close()


def test_oversize_refused(local8):
    K, progs = golden_programs("cfg1")
    with pytest.raises(ExecError) as e:
        local8.compile(progs[0][2], (256 << 20) // 4 + 1, "f32")
    assert e.value.code == 3


# ---- several GPUs, one process --------------------------------------------

@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("mapping", ["block", "interleave"])
@pytest.mark.parametrize("push", [False, True])
def test_two_gpus_config2(mapping, push):
    ords = [d * 2 // 8 for d in range(8)] if mapping == "block" else [d % 2 for d in range(8)]
    ctx = executor.Context.local(8, ords, max_bytes=64 << 20)
    ctx.set_option("push_min_bytes", 0 if push else -1)
    try:
        for name in ("cfg2_r1", "cfg2_r01"):
            K, progs = golden_programs(name)
            for _, _, prog, _ in progs[::3]:
                _run(ctx, prog, K, 3001, numeric.BF16)
        K, progs = golden_programs("cfg2_r01")
        for _, _, prog, _ in progs[::100]:
            _run(ctx, prog, K, 8 << 20, numeric.BF16, runs=2)
    finally:
        ctx.close()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("push,ll", [(False, False), (True, False), (False, True)])
def test_one_slot_per_gpu_small_k(push, ll):
    n = min(NGPU, 8)
    name = {2: "k2_flat", 4: "k4_sock", 8: "k8_sock"}.get(n)
    if name is None:
        pytest.skip("GPU count without a golden set")
    ctx = executor.Context.local(n, list(range(n)), max_bytes=64 << 20)
    ctx.set_option("push_min_bytes", 0 if push else -1)
    ctx.set_option("ll_max_bytes", (256 << 10) if ll else 0)
    ctx.set_option("ll_total_bytes", 3 << 20)
    try:
        K, progs = golden_programs(name)
        for _, _, prog, _ in progs:
            _run(ctx, prog, K, 4097, numeric.F32)
        for _, _, prog, _ in progs[:4]:
            _run(ctx, prog, K, 16 << 20, numeric.BF16, runs=3)
    finally:
        ctx.close()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_one_shot_steps_repeated():
    """One-shot (LL) steps: packets alternate between two parity regions by
    epoch, so many back-to-back runs must chain exactly; ragged sizes exercise
    the edge packets; every dtype bit-exact. (Graph replay of one-shot steps:
    test_gpu_multiprocess.py, one process per GPU.)"""
    n = min(NGPU, 8)
    name = {2: "k2_flat", 4: "k4_sock", 8: "k8_sock"}.get(n)
    if name is None:
        pytest.skip("GPU count without a golden set")
    ctx = executor.Context.local(n, list(range(n)), max_bytes=8 << 20)
    ctx.set_option("ll_total_bytes", 3 << 20)
    try:
        K, progs = golden_programs(name)
        for N in (1, 13, 1001, 32 << 10):
            for dt in (numeric.BF16, numeric.F32, numeric.I32):
                for _, _, prog, _ in progs[:6]:
                    plan = ctx.compile(prog, N, dt)
                    assert all(plan.describe()["phase_ll"])
                    plan.close()
                    _run(ctx, prog, K, N, dt, runs=5)
    finally:
        ctx.close()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
@pytest.mark.parametrize("ll", [False, True])
def test_config3_programs_across_gpus(ll):
    """Config 3 (axes [2,2,2], every one- and two-axis request) with the 8
    slots block-distributed over the GPUs; one-shot steps on or off."""
    n = min(NGPU, 4)
    ctx = executor.Context.local(8, [d * n // 8 for d in range(8)], max_bytes=8 << 20)
    ctx.set_option("ll_max_bytes", (256 << 10) if ll else 0)
    ctx.set_option("ll_total_bytes", 3 << 20)
    try:
        for name in ("cfg3_r0", "cfg3_r1", "cfg3_r2", "cfg3_r01", "cfg3_r02", "cfg3_r12"):
            K, progs = golden_programs(name)
            for _, _, prog, _ in progs[::9]:
                _run(ctx, prog, K, 1001, numeric.F32)
                _run(ctx, prog, K, 777, numeric.I32, runs=2)
    finally:
        ctx.close()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_config1_full_size_across_gpus():
    """Config 1 at its full size (64 MiB f32 per device) on 2 or 4 GPUs."""
    n = min(NGPU, 4)
    ctx = executor.Context.local(8, [d * n // 8 for d in range(8)], max_bytes=64 << 20)
    try:
        K, progs = golden_programs("cfg1")
        N = 16 * 1024 * 1024
        inputs = numeric.synthetic_inputs(K, N, numeric.F32)
        for _, _, prog, _ in progs:
            _run(ctx, prog, K, N, numeric.F32, inputs=inputs)
    finally:
        ctx.close()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 2, reason="needs >= 2 GPUs")
def test_interleaved_variants_share_epochs():
    """Plans of different variants (one-shot single step, one-shot two-step
    with the relaxed wait, pull, push) share one context's epochs and LL
    parity regions: run them interleaved many times, in place, and compare
    with the oracle applied in the same order."""
    n = min(NGPU, 8)
    name = {2: "k2_flat", 4: "k4_sock", 8: "k8_sock"}.get(n)
    if name is None:
        pytest.skip("GPU count without a golden set")
    K, progs = golden_programs(name)
    ctx = executor.Context.local(n, list(range(n)), max_bytes=8 << 20)
    ctx.set_option("ll_total_bytes", 3 << 20)
    try:
        single = progs[0][2]
        multi = next(p for _, _, p, _ in progs if len(p.steps) >= 2)
        N_small, N_big = 3001, (1 << 20) + 5
        plans = [(single, N_small), (multi, N_small), (single, N_big), (multi, N_big)]
        compiled = []
        for i, (prog, N) in enumerate(plans):
            ctx.set_option("push_min_bytes", 0 if i == 3 else -1)
            compiled.append(ctx.compile(prog, N, "i32"))
        assert compiled[0].describe()["phase_ll"] == [1]
        assert all(compiled[1].describe()["phase_ll"])
        assert not any(compiled[2].describe()["phase_ll"])
        inputs = numeric.synthetic_inputs(K, N_big, numeric.I32)
        for d in range(K):
            ctx.write(d, inputs[d])
        want = [x.copy() for x in inputs]
        order = [0, 1, 0, 2, 1, 1, 3, 0, 2, 3, 1, 0, 0, 2, 1, 3] * 3
        for i in order:
            compiled[i].run()
            prog, N = plans[i]
            head = [x[:N].copy() for x in want]
            numeric.execute(prog, K, head, numeric.I32)
            for d in range(K):
                want[d][:N] = head[d]
        ctx.synchronize()
        for d in range(K):
            assert np.array_equal(ctx.read(d, N_big * 4), want[d].view(np.uint8)), d
        for p in compiled:
            p.close()
    finally:
        ctx.close()


@pytest.mark.multigpu
@pytest.mark.skipif(NGPU < 3, reason="needs >= 3 GPUs")
def test_three_gpus_shuffled_slots_every_variant():
    """8 slots shuffled over 3 GPUs (uneven, non power of two): one-shot,
    pull and push steps, bit-exact."""
    import random
    rng = random.Random(3)
    ords = [d % 3 for d in range(8)]
    rng.shuffle(ords)
    ctx = executor.Context.local(8, ords, max_bytes=16 << 20)
    try:
        K, progs = golden_programs("cfg2_r01")
        for _, _, prog, _ in progs[::60]:
            _run(ctx, prog, K, 3001, numeric.BF16, runs=2)
        ctx.set_option("push_min_bytes", 0)
        for _, _, prog, _ in progs[::90]:
            _run(ctx, prog, K, (4 << 20) - 3, numeric.I32, runs=2)
    finally:
        ctx.close()


def test_cpp_host_example_end_to_end():
    """C++ host: reference planner API -> redsynth::GpuExecutor::Execute on
    every config-2 (reduce {0,1}) program, int32 identity checked in C++."""
    import subprocess
    from common import ROOT
    exe = os.path.join(ROOT, "paper_2110_10548_b200", "_lib", "execute_example")
    r = subprocess.run([exe, os.path.join(ROOT, "configs", "b200_sock.json"), "2,4", "0,1", "4099"],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "programs=500 mismatches=0" in r.stdout
    assert "step 1: Reduce over devices {0,1}: devices hold different chunk sets" in r.stdout


def test_synth_cli_execute_mode(tmp_path):
    """`synth --execute`: the reference report plus measured columns."""
    import json
    import subprocess
    from common import ROOT
    exe = os.path.join(ROOT, "paper_2110_10548_b200", "_lib", "synth")
    out = tmp_path / "r.json"
    r = subprocess.run([exe, "--system", os.path.join(ROOT, "configs", "b200_sock.json"), "--axes", "2,4",
                        "--reduce", "0", "--bytes", str(8 << 20), "--execute", "--iters", "3", "--out", str(out)],
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr
    doc = json.loads(out.read_text())
    assert doc["executed"]["dtype"] == "bf16"
    for m in doc["matrices"]:
        assert m["measured_best"]["us"] > 0
        ranks = sorted(p["measured_rank"] for p in m["programs"])
        assert ranks == list(range(1, len(m["programs"]) + 1))
        assert m["calibrated_best"]["measured_us"] > 0
        for p in m["programs"]:
            assert p["measured_us"] > 0 and p["bus_GBps"] > 0 and p["calibrated_us"] > 0
