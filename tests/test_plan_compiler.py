"""The executor's plan compiler on CPU (planning-only contexts, no GPU).

Every compiled plan is executed by a numpy simulator of the step kernel's
contract (tests/common.py::simulate_plan), which first proves the step's
tasks hazard-free (no byte written by one task is touched by another), and
the result must equal the C oracle bit for bit — for every synthesized
program of the baseline configs, several slot->GPU mappings, and ragged
sizes. Barrier sets are checked against an independent derivation.
"""
import json
import os
import random

import numpy as np
import pytest

from common import GOLDEN, golden_programs, simulate_plan
from oracle import numeric
from paper_2110_10548_b200 import executor
from paper_2110_10548_b200._native import ExecError

MAPPINGS = {
    "local": lambda K: ([0] * K, 1),
    "two_gpus": lambda K: ([d * 2 // K for d in range(K)], 2),
    "four_gpus": lambda K: ([d * 4 // K for d in range(K)], 4),
    "one_per_gpu": lambda K: (list(range(K)), K),
    "interleaved2": lambda K: ([d % 2 for d in range(K)], 2),
}


def _compile(prog, K, mapping, N, dtype, push=False, ll=False):
    slot_rank, world = MAPPINGS[mapping](K)
    ctx = executor.Context.virtual(K, slot_rank, world)
    ctx.set_option("push_min_bytes", 0 if push else -1)
    if world > 1:
        ctx.set_option("ll_max_bytes", (256 << 10) if ll else 0)
        ctx.set_option("ll_total_bytes", 3 << 20)
    plan = ctx.compile(prog, N, dtype)
    return ctx, plan, plan.describe()


def _check(prog, K, mapping, N, dtype, push=False, ll=False):
    ctx, plan, desc = _compile(prog, K, mapping, N, dtype, push, ll)
    inputs = numeric.synthetic_inputs(K, N, dtype)
    want = [x.copy() for x in inputs]
    numeric.execute(prog, K, want, dtype, nthreads=1)
    got = [x.copy() for x in inputs]
    simulate_plan(desc, got, dtype)
    for d in range(K):
        assert np.array_equal(got[d].view(np.uint8), want[d].view(np.uint8)), (prog.text, mapping, d)
    return desc


@pytest.mark.parametrize("name", ["cfg1", "cfg2_r1", "cfg2_r01"])
def test_every_program_bit_exact_bf16_one_per_gpu(name):
    K, progs = golden_programs(name)
    for _, _, prog, _ in progs:
        _check(prog, K, "one_per_gpu", 333, numeric.BF16)


@pytest.mark.parametrize("name", ["cfg3_r0", "cfg3_r1", "cfg3_r2", "cfg3_r01", "cfg3_r02", "cfg3_r12"])
def test_every_config3_program_bit_exact_f32(name):
    K, progs = golden_programs(name)
    for _, _, prog, _ in progs:
        _check(prog, K, "one_per_gpu", 61, numeric.F32)


@pytest.mark.parametrize("mapping", ["local", "two_gpus", "four_gpus", "interleaved2"])
@pytest.mark.parametrize("dtype", [numeric.F32, numeric.BF16, numeric.I32])
def test_sampled_programs_other_mappings(mapping, dtype):
    rng = random.Random(7)
    for name in ("cfg2_r01", "cfg2_r1", "cfg3_r12", "k8_sock"):
        K, progs = golden_programs(name)
        for _, _, prog, _ in rng.sample(progs, min(25, len(progs))):
            _check(prog, K, mapping, rng.choice([8, 15, 64, 257, 1000, 4099]), dtype)


@pytest.mark.parametrize("name", ["cfg1", "cfg2_r1", "cfg2_r01", "k8_sock"])
@pytest.mark.parametrize("mapping", ["two_gpus", "interleaved2"])
def test_push_variant_every_program_bit_exact(name, mapping):
    """Push variant between two GPUs (one launch: sources land the owners'
    parts in their scratch chunk by chunk behind flags, owners reduce each
    landed chunk and push the results): same bits as the oracle,
    hazard-free, and in AllReduce steps no vector task reads memory of
    another GPU (only < 16-byte edges pull)."""
    K, progs = golden_programs(name)
    for _, _, prog, _ in progs[:: 2 if name.startswith("cfg2") else 1]:
        desc = _check(prog, K, mapping, 517, numeric.BF16, push=True)
        assert desc["num_phases"] == len(prog.steps)  # one launch per step
        for step, (op, _) in zip(desc["steps"], prog.steps):
            if op != 0:  # RS / Reduce / one-to-all copies pull (measured faster)
                continue
            for r, rk in enumerate(step["ranks"]):
                for t in rk["tasks"]:
                    if t["vec"]:
                        assert all(desc["slot_rank"][s] == r for s in t["src"]), (prog.text, t)


def test_push_senders_rotate_targets():
    """With several GPUs pushing, each sender walks the receiving GPUs
    starting after itself (GPU r lands in r+1, r+2, ...), so the GPUs push
    into different peers at any moment instead of all into one (incast)."""
    K, progs = golden_programs("k4_flat")
    _, _, desc = _compile(progs[0][2], K, "one_per_gpu", 1 << 20, numeric.F32, push=True)
    for r, rk in enumerate(desc["steps"][0]["ranks"]):
        targets = [t["dst"][0] for t in rk["tasks"] if t["mode"] == 3]
        assert targets == [(r + k) % K for k in range(1, K)], (r, targets)


@pytest.mark.parametrize("mapping", ["two_gpus", "four_gpus", "interleaved2"])
@pytest.mark.parametrize("dtype", [numeric.F32, numeric.I32])
def test_push_variant_other_mappings(mapping, dtype):
    rng = random.Random(11)
    for name in ("cfg2_r01", "cfg3_r02", "cfg3_r12"):
        K, progs = golden_programs(name)
        for _, _, prog, _ in rng.sample(progs, min(40, len(progs))):
            _check(prog, K, mapping, rng.choice([9, 64, 1003, 4099]), dtype, push=True)


def test_push_allreduce_traffic_is_store_only():
    K, progs = golden_programs("k2_flat")
    prog = progs[0][2]
    _, plan, desc = _compile(prog, K, "one_per_gpu", 1 << 20, numeric.BF16, push=True)
    assert desc["num_phases"] == 1 and desc["phase_step"] == [0]
    modes = {t["mode"] for rk in desc["steps"][0]["ranks"] for t in rk["tasks"]}
    assert modes <= {0, 3, 4} and {3, 4} <= modes
    link, _ = plan.step_bytes(0)
    D = (1 << 20) * 2
    assert abs(link - 2 * 1 / 2 * D) <= 256  # same 2(n-1)/n D per direction, all stores


@pytest.mark.parametrize("N", [0, 1, 5, 8, 9, 31, 127])
def test_ragged_and_tiny_sizes(N):
    K, progs = golden_programs("cfg2_r01")
    for _, _, prog, _ in progs[::20]:
        _check(prog, K, "one_per_gpu", N, numeric.BF16)
        _check(prog, K, "local", N, numeric.I32)


def test_small_k_sets():
    for name in ("k2_flat", "k4_flat", "k4_sock", "k8_flat"):
        K, progs = golden_programs(name)
        for _, _, prog, _ in progs:
            for mapping in ("local", "one_per_gpu"):
                _check(prog, K, mapping, 1001, numeric.F32)


def _group_of(prog, s, d):
    if s < 0:
        return [d]
    for g in prog.steps[s][1]:
        if d in g:
            return g
    return [d]


def test_barrier_sets_match_independent_derivation():
    K, progs = golden_programs("cfg2_r01")
    for mapping in ("one_per_gpu", "two_gpus", "interleaved2"):
        slot_rank, world = MAPPINGS[mapping](K)
        for _, _, prog, _ in progs[::7]:
            _, _, desc = _compile(prog, K, mapping, 100, numeric.F32)
            for s, step in enumerate(desc["steps"]):
                for r, rk in enumerate(step["ranks"]):
                    expect = set()
                    for d in range(K):
                        if slot_rank[d] != r:
                            continue
                        for q in _group_of(prog, s, d):
                            for p in _group_of(prog, s - 1, q):
                                expect.add(slot_rank[p])
                    expect.discard(r)
                    assert set(rk["wait"]) == expect
            for r in range(world):
                expect = {slot_rank[p] for d in range(K) if slot_rank[d] == r
                          for p in _group_of(prog, len(prog.steps) - 1, d)} - {r}
                assert set(desc["final_wait"][r]) == expect


def test_allreduce_is_one_pass_two_shot():
    """Baseline AllReduce over n members: each owner reduces a 1/n slice
    (16-byte aligned cut points) and pushes it to all n members."""
    K, progs = golden_programs("cfg2_r01")
    prog = progs[0][2]
    assert prog.text == "Slice(root) InsideGroup AllReduce"
    _, plan, desc = _compile(prog, K, "one_per_gpu", 1 << 20, numeric.BF16)
    step = desc["steps"][0]
    sizes = [sum(t["hi"] - t["lo"] for t in rk["tasks"]) for rk in step["ranks"]]
    assert max(sizes) - min(sizes) <= 16
    for rk in step["ranks"]:
        for t in rk["tasks"]:
            assert len(t["src"]) == 8 and len(t["dst"]) == 8
    link, _ = plan.step_bytes(0)
    D = (1 << 20) * 2
    assert abs(link - 2 * 7 / 8 * D) <= 64  # 2(n-1)/n D per direction


def test_broadcast_relay_balances_root_link():
    """Reduce -> Broadcast over 8: the root sends each byte once (relay by
    the receivers), so its per-direction traffic is ~1 x D, not 7 x D."""
    K, progs = golden_programs("k8_flat")
    prog = next(p for _, _, p, _ in progs if p.text.endswith("Reduce; Slice(root) InsideGroup Broadcast"))
    _, plan, desc = _compile(prog, K, "one_per_gpu", 1 << 20, numeric.F32)
    D = (1 << 20) * 4
    for s in range(2):
        link, _ = plan.step_bytes(s)
        assert link <= 1.01 * D, (s, link / D)


def test_refusals_match_reference():
    from paper_2110_10548_b200.planner import LoweredProgram
    cases = json.load(open(os.path.join(GOLDEN, "refusals.json")))
    ctx = executor.Context.virtual(8, list(range(8)), 8)
    for c in cases:
        prog = LoweredProgram(steps=[(op, gs) for op, gs in c["steps"]])
        if c["code"] == 0:
            ctx.compile(prog, 64, "f32")
            continue
        with pytest.raises(ExecError) as e:
            ctx.compile(prog, 64, "f32")
        assert e.value.code == c["code"] and e.value.message == c["message"]


def test_structural_refusals():
    from paper_2110_10548_b200.planner import LoweredProgram
    ctx = executor.Context.virtual(4, [0, 1, 2, 3], 4)
    with pytest.raises(ExecError) as e:
        ctx.compile(LoweredProgram(steps=[(0, [])]), 8)
    assert e.value.code == 3 and e.value.message == "step 0 has no device groups"
    with pytest.raises(ExecError) as e:  # out of range -> reference violation name
        ctx.compile(LoweredProgram(steps=[(0, [[0, 9]])]), 8)
    assert e.value.code == 9 and "device outside the state context" in e.value.message
    with pytest.raises(ExecError) as e:  # groups not disjoint: executor precondition
        ctx.compile(LoweredProgram(steps=[(2, [[0, 1], [1, 2]])]), 8)
    assert e.value.code in (3, 9)
    with pytest.raises(ExecError) as e:
        ctx.compile(LoweredProgram(steps=[(7, [[0, 1]])]), 8)
    assert e.value.code == 3
    # an empty program is a valid no-op (RunLowered returns the initial state)
    ctx.compile(LoweredProgram(steps=[]), 8)


def test_nvls_plan_structure_virtual():
    """With NVLS on, AllReduce groups of >= 4 slots on distinct GPUs become
    multicast tasks (one per owner slice); smaller groups and int32 stay P2P.
    The plan stays hazard-free (simulated with ordered sums)."""
    K, progs = golden_programs("cfg2_r01")
    ctx = executor.Context.virtual(K, list(range(K)), K)
    ctx.set_option("push_min_bytes", -1)
    ctx.set_option("nvls", 1)
    ctx.set_option("nvls_min_bytes", 0)
    ctx.set_option("ll_max_bytes", 0)  # one-shot would take these small steps
    seen = 0
    for _, _, prog, _ in progs[::10]:
        for dtype in (numeric.BF16, numeric.I32):
            plan = ctx.compile(prog, 4099, dtype)
            desc = plan.describe()
            for st, (op, groups) in zip(desc["steps"], prog.steps):
                for rk in st["ranks"]:
                    for t in rk["tasks"]:
                        if t.get("mode") == 1:
                            seen += 1
                            assert dtype != numeric.I32 and op == 0 and len(t["src"]) >= 4
            inputs = numeric.synthetic_inputs(K, 4099, dtype)
            want = [x.copy() for x in inputs]
            numeric.execute(prog, K, want, dtype, nthreads=1)
            got = [x.copy() for x in inputs]
            simulate_plan(desc, got, dtype)
            assert all(np.array_equal(a.view(np.uint8), b.view(np.uint8)) for a, b in zip(got, want))
    assert seen > 0


# ---- one-shot (LL) steps ----------------------------------------------------

@pytest.mark.parametrize("name", ["cfg1", "cfg2_r1", "cfg2_r01", "k8_sock", "k4_flat", "k2_flat"])
@pytest.mark.parametrize("dtype", [numeric.F32, numeric.BF16, numeric.I32])
def test_ll_every_program_bit_exact_one_per_gpu(name, dtype):
    """Small buffers, one slot per GPU: every step is one-shot, the plan is
    hazard-free, every packet stream has a sender, and the bits equal the
    oracle's (each destination sums all members in group order)."""
    K, progs = golden_programs(name)
    for _, _, prog, _ in progs[:: 3 if name.startswith("cfg2") else 1]:
        desc = _check(prog, K, "one_per_gpu", 333, dtype, ll=True)
        assert all(desc["phase_ll"]), prog.text
        assert desc["final_wait"] == [[] for _ in range(K)]
        # one-shot after one-shot waits one epoch less; the last phase's
        # epoch is never awaited
        assert desc["phase_lag"] == [0] + [1] * (desc["num_phases"] - 1)
        assert not any(rk["signal"] for rk in desc["steps"][-1]["ranks"])
        for step in desc["steps"]:
            for r, rk in enumerate(step["ranks"]):
                for t in rk["tasks"]:
                    # no task addresses another GPU's slot buffer directly
                    assert all(desc["slot_rank"][x] == r for x, rg in zip(t["src"], t["src_region"]) if rg == -1)
                    assert all(desc["slot_rank"][x] == r for x in t["dst"])


@pytest.mark.parametrize("mapping", ["two_gpus", "four_gpus", "interleaved2"])
@pytest.mark.parametrize("dtype", [numeric.BF16, numeric.I32])
def test_ll_mixed_mappings(mapping, dtype):
    """Several slots per GPU: steps whose cross-GPU groups have one member per
    GPU run one-shot (GPU-local groups as ordinary tasks in the same launch),
    the others fall back to the pull path; bits equal the oracle's."""
    rng = random.Random(5)
    seen = 0
    for name in ("cfg2_r01", "cfg2_r1", "cfg3_r12", "k8_sock"):
        K, progs = golden_programs(name)
        for _, _, prog, _ in rng.sample(progs, min(25, len(progs))):
            desc = _check(prog, K, mapping, rng.choice([8, 15, 64, 257, 1000, 4099]), dtype, ll=True)
            seen += sum(desc["phase_ll"])
    assert seen > 0


@pytest.mark.parametrize("N", [0, 1, 5, 9, 31, 127, 4097])
def test_ll_ragged_sizes(N):
    K, progs = golden_programs("cfg2_r01")
    for _, _, prog, _ in progs[::25]:
        _check(prog, K, "one_per_gpu", N, numeric.BF16, ll=True)


def test_ll_budget_selects_variant():
    """An AllReduce of D bytes over n GPUs sends D to each peer: one-shot at
    D <= ll_max_bytes per peer and (n-1) D <= ll_total_bytes per sender,
    pull above. Defaults: 256 KiB per peer, 16 KiB per sender."""
    K, progs = golden_programs("k4_flat")
    prog = progs[0][2]
    ctx = executor.Context.virtual(K, list(range(K)), K)
    ctx.set_option("push_min_bytes", -1)
    D = (16 << 10) // 3 // 8 * 8  # default total cap, 3 peers
    assert ctx.compile(prog, D // 4, "f32").describe()["phase_ll"] == [1]
    assert ctx.compile(prog, (D + 64) // 4, "f32").describe()["phase_ll"] == [0]
    ctx.set_option("ll_total_bytes", 3 << 20)
    ctx.set_option("ll_max_bytes", 64 << 10)
    assert ctx.compile(prog, (64 << 10) // 4, "f32").describe()["phase_ll"] == [1]
    assert ctx.compile(prog, (64 << 10) // 4 + 2, "f32").describe()["phase_ll"] == [0]
    ctx.set_option("ll_max_bytes", 0)
    assert ctx.compile(prog, 16, "f32").describe()["phase_ll"] == [0]
    ctx.set_option("ll_max_bytes", 1 << 30)  # capped by the reserved area (512 KiB)
    assert ctx.compile(prog, (1 << 20) // 4, "f32").describe()["phase_ll"] == [0]
    K, progs = golden_programs("k8_flat")  # 7 peers: the per-sender cap binds first
    ctx = executor.Context.virtual(K, list(range(K)), K)
    ctx.set_option("ll_max_bytes", 64 << 10)
    ctx.set_option("ll_total_bytes", 3 * (64 << 10))
    D = 3 * (64 << 10) // 7 // 8 * 8
    assert ctx.compile(progs[0][2], D // 4, "f32").describe()["phase_ll"] == [1]
    assert ctx.compile(progs[0][2], (D + 64) // 4, "f32").describe()["phase_ll"] == [0]


def test_ll_allreduce_sends_from_inside_the_owner_task():
    """One-shot AllReduce: each GPU's single task reads its slot, sends it to
    the 7 peers and sums the 8 packet streams in group order (no separate
    send tasks, so the value sent is read before it is overwritten)."""
    K, progs = golden_programs("k8_flat")
    prog = progs[0][2]
    _, plan, desc = _compile(prog, K, "one_per_gpu", 1000, numeric.F32, ll=True)
    for r, rk in enumerate(desc["steps"][0]["ranks"]):
        assert len(rk["tasks"]) == 1
        t = rk["tasks"][0]
        assert t["mode"] == 2 and t["dst"] == [r] and sorted(t["sends"]) == [q for q in range(8) if q != r]
        assert t["src"] == list(range(8))
        assert [rg for rg in t["src_region"]] == [-1 if x == r else -3 for x in range(8)]


def test_calibrated_cost_model():
    """rs_plan_predict_us: per launch, latency + the plan's own max link bytes
    / link rate + max HBM bytes / HBM rate."""
    K, progs = golden_programs("k8_flat")
    prog = progs[0][2]  # single AllReduce over 8 GPUs
    N = 1 << 24  # f32, 64 MiB per GPU
    _, plan, desc = _compile(prog, K, "one_per_gpu", N, numeric.F32)
    link, hbm = plan.step_bytes(0)
    us = plan.predict_us(launch_us=8.0, link_gbs=650.0, hbm_gbs=6000.0)
    assert abs(us - (8.0 + link / 650e3 + hbm / 6000e3)) < 1e-6
    assert abs(link - 2 * 7 / 8 * N * 4) <= 64
    # one GPU: no link bytes, the HBM term only
    _, plan1, _ = _compile(prog, K, "local", N, numeric.F32)
    l1, h1 = plan1.step_bytes(0)
    assert l1 == 0 and abs(plan1.predict_us(3.0, 650.0, 6000.0) - (3.0 + h1 / 6000e3)) < 1e-6
    with pytest.raises(ExecError):
        plan.predict_us(8.0, 0.0, 6000.0)


@pytest.mark.parametrize("seed", range(6))
def test_random_slot_to_gpu_mappings(seed):
    """Arbitrary slot -> GPU maps (3, 5, 6, 7 GPUs, slots shuffled) under
    every variant threshold setting: hazard-free and bit-exact."""
    rng = random.Random(100 + seed)
    world = [3, 5, 6, 7, 2, 4][seed]
    for name in ("cfg2_r01", "cfg3_r12", "k8_sock"):
        K, progs = golden_programs(name)
        slot_rank = [d % world for d in range(K)]
        rng.shuffle(slot_rank)
        for _, _, prog, _ in rng.sample(progs, min(12, len(progs))):
            for push, ll in ((False, False), (True, False), (False, True)):
                ctx = executor.Context.virtual(K, slot_rank, world)
                ctx.set_option("push_min_bytes", 0 if push else -1)
                ctx.set_option("ll_max_bytes", (256 << 10) if ll else 0)
                ctx.set_option("ll_total_bytes", 3 << 20)
                N = rng.choice([7, 100, 2049, 5000])
                dtype = rng.choice([numeric.F32, numeric.BF16, numeric.I32])
                desc = ctx.compile(prog, N, dtype).describe()
                inputs = numeric.synthetic_inputs(K, N, dtype)
                want = [x.copy() for x in inputs]
                numeric.execute(prog, K, want, dtype, nthreads=1)
                got = [x.copy() for x in inputs]
                simulate_plan(desc, got, dtype)
                for d in range(K):
                    assert np.array_equal(got[d].view(np.uint8), want[d].view(np.uint8)), (prog.text, slot_rank, d)


def test_two_member_reduce_is_pulled_by_the_root():
    """Reduce over 2 GPUs: the root pulls the other member's data and sums
    locally, so the link carries D one way only; wider groups keep
    non-root owners (~D per direction on every GPU)."""
    from paper_2110_10548_b200.planner import LoweredProgram
    ctx = executor.Context.virtual(2, [0, 1], 2)
    ctx.set_option("ll_max_bytes", 0)
    plan = ctx.compile(LoweredProgram(steps=[(3, [[0, 1]])]), 1 << 20, "f32")
    desc = plan.describe()
    assert desc["steps"][0]["ranks"][1]["tasks"] == []
    assert all(t["dst"] == [0] and t["src"] == [0, 1] for t in desc["steps"][0]["ranks"][0]["tasks"])
    rk0, rk1 = desc["steps"][0]["ranks"]
    assert rk0["rx"] == 4 << 20 and rk0["tx"] == 0 and rk1["tx"] == 4 << 20


def test_copies_push_only_when_balanced():
    """AllGather after a ReduceScatter (every member holds a run) pushes;
    AllGather / Broadcast from a single holder (after a Reduce) pulls."""
    K, progs = golden_programs("k2_flat")
    rs_ag = next(p for _, _, p, _ in progs if p.text.startswith("Slice(root) InsideGroup ReduceScatter"))
    red_bc = next(p for _, _, p, _ in progs if p.text.endswith("Broadcast"))
    _, _, d1 = _compile(rs_ag, K, "one_per_gpu", 1 << 20, numeric.F32, push=True)
    _, _, d2 = _compile(red_bc, K, "one_per_gpu", 1 << 20, numeric.F32, push=True)
    modes = lambda d, s: {t["mode"] for rk in d["steps"][s]["ranks"] for t in rk["tasks"]}  # noqa: E731
    assert 3 in modes(d1, 1)
    assert modes(d2, 1) <= {0}


@pytest.mark.parametrize("mode", [1, 2, 3, 4])
@pytest.mark.parametrize("mapping", ["one_per_gpu", "four_gpus"])
def test_reduce_modes_bit_exact_and_shaped(mode, mapping):
    """Reduce over >= 3 GPUs (semantics.cc:292-299): push (mode 1, store-only
    landing behind chunk flags) and NVLS (mode 2: every member owns a slice;
    mode 3: the root owns all) — hazard-free plans whose ordered-sum
    simulation equals the oracle; NVLS tasks only where a group has one slot
    per GPU and the data is floating point."""
    K, progs = golden_programs("cfg2_r01")
    slot_rank, world = MAPPINGS[mapping](K)
    ctx = executor.Context.virtual(K, slot_rank, world)
    ctx.set_option("ll_max_bytes", 0)
    ctx.set_option("push_min_bytes", 0)
    ctx.set_option("reduce_mode", mode)
    if mode >= 2:
        ctx.set_option("nvls", 1)
        ctx.set_option("nvls_min_bytes", 0)
    reduce_progs = [p for _, _, p, _ in progs if any(op == 3 for op, _ in p.steps)]
    seen = 0
    for prog in reduce_progs[::7]:
        for dtype in (numeric.BF16, numeric.I32):
            desc = ctx.compile(prog, 4099, dtype).describe()
            for st, (op, groups) in zip(desc["steps"], prog.steps):
                if op != 3:
                    continue
                for rk in st["ranks"]:
                    for t in rk["tasks"]:
                        if t.get("mode") == 5:
                            seen += 1
                            assert mode >= 2 and dtype != numeric.I32
                            assert len(t["src"]) >= 4 and len(t["dst"]) == 1 and t["dst"][0] == t["src"][0]
                        if mode in (1, 4) and t.get("mode") in (3, 4):
                            seen += 1
            inputs = numeric.synthetic_inputs(K, 4099, dtype)
            want = [x.copy() for x in inputs]
            numeric.execute(prog, K, want, dtype, nthreads=1)
            got = [x.copy() for x in inputs]
            simulate_plan(desc, got, dtype)
            assert all(np.array_equal(a.view(np.uint8), b.view(np.uint8)) for a, b in zip(got, want)), prog.text
    if mapping == "one_per_gpu" or mode in (1, 4):
        assert seen > 0


def test_reduce_mode_option_validated():
    ctx = executor.Context.virtual(4, [0, 1, 2, 3], 4)
    with pytest.raises(ExecError):
        ctx.set_option("reduce_mode", 7)
    with pytest.raises(ExecError):
        ctx.set_option("reduce_mode", -2)


def test_reduce_auto_policy_by_size():
    """Default Reduce policy (reduce_mode -1): groups of >= 3 members pull
    below reduce_push_min_bytes and push (waves) from there; 2-member groups
    are always pulled by the root."""
    from paper_2110_10548_b200.planner import LoweredProgram
    ctx = executor.Context.virtual(4, [0, 1, 2, 3], 4)
    ctx.set_option("ll_max_bytes", 0)
    ctx.set_option("reduce_push_min_bytes", 1 << 20)
    prog = LoweredProgram(steps=[(3, [[0, 1, 2, 3]])])
    small = ctx.compile(prog, (1 << 19) // 2, numeric.BF16).describe()
    big = ctx.compile(prog, (4 << 20) // 2, numeric.BF16).describe()
    modes = lambda d: {t["mode"] for rk in d["steps"][0]["ranks"] for t in rk["tasks"]}
    assert modes(small) == {0}
    assert {3, 4} <= modes(big)
    ctx.set_option("reduce_mode", 0)
    assert modes(ctx.compile(prog, (4 << 20) // 2, numeric.BF16).describe()) == {0}


@pytest.mark.parametrize("lag", [0, 2])
@pytest.mark.parametrize("mapping", ["one_per_gpu", "two_gpus", "interleaved2"])
@pytest.mark.parametrize("reduce_mode", [0, 1])
def test_push_waves_bit_exact_and_ordered(mapping, reduce_mode, lag):
    """Push waves (push_wave_bytes): parts are cut into waves whose landing
    tasks precede their reducing tasks (by wave_lag waves) — the plan stays
    hazard-free and equal to the oracle; unaligned part edges still pull
    (scalar tasks only at the true edges)."""
    K, progs = golden_programs("cfg2_r01")
    slot_rank, world = MAPPINGS[mapping](K)
    ctx = executor.Context.virtual(K, slot_rank, world)
    ctx.set_option("ll_max_bytes", 0)
    ctx.set_option("push_min_bytes", 0)
    ctx.set_option("push_wave_bytes", 16 << 10)
    ctx.set_option("reduce_wave_bytes", 16 << 10)
    ctx.set_option("reduce_mode", reduce_mode)
    ctx.set_option("wave_lag", lag)
    N = (1 << 17) + 3
    waves = 0
    for _, _, prog, _ in progs[::23]:
        desc = ctx.compile(prog, N, numeric.BF16).describe()
        for st in desc["steps"]:
            for rk in st["ranks"]:
                modes = [t["mode"] for t in rk["tasks"]]
                sends = [i for i, m in enumerate(modes) if m == 3]
                recvs = [i for i, m in enumerate(modes) if m == 4]
                if len(sends) > 1:
                    waves += 1
                # interleaved: some reducing task precedes the last landing task
                if len(sends) > 4 and recvs and lag == 0:
                    assert recvs[0] < sends[-1], modes
                assert sum(1 for t in rk["tasks"] if not t["vec"]) <= 4 * len(rk["tasks"])
        inputs = numeric.synthetic_inputs(K, N, numeric.BF16)
        want = [x.copy() for x in inputs]
        numeric.execute(prog, K, want, numeric.BF16, nthreads=1)
        got = [x.copy() for x in inputs]
        simulate_plan(desc, got, numeric.BF16)
        assert all(np.array_equal(a.view(np.uint8), b.view(np.uint8)) for a, b in zip(got, want)), prog.text
    assert waves > 0


def test_nvls_broadcast_plan_virtual():
    """With NVLS on, Broadcast groups on distinct GPUs whose members all need
    every row become one multicast store stream from the root (mode 6, any
    dtype); the ordered simulation equals the oracle bit for bit."""
    K, progs = golden_programs("k4_sock")
    ctx = executor.Context.virtual(K, list(range(K)), K)
    ctx.set_option("nvls", 1)
    ctx.set_option("nvls_bcast", 1)
    ctx.set_option("nvls_min_bytes", 0)
    ctx.set_option("ll_max_bytes", 0)
    seen = 0
    for _, _, prog, _ in progs:
        if not any(op == 4 for op, _ in prog.steps):
            continue
        for dtype in (numeric.I32, numeric.BF16):
            desc = ctx.compile(prog, 4099, dtype).describe()
            for st, (op, groups) in zip(desc["steps"], prog.steps):
                for rk in st["ranks"]:
                    for t in rk["tasks"]:
                        if t.get("mode") == 6:
                            seen += 1
                            assert op == 4 and len(t["src"]) == 1 and len(t["dst"]) == len(groups[0]) - 1
            inputs = numeric.synthetic_inputs(K, 4099, dtype)
            want = [x.copy() for x in inputs]
            numeric.execute(prog, K, want, dtype, nthreads=1)
            got = [x.copy() for x in inputs]
            simulate_plan(desc, got, dtype)
            assert all(np.array_equal(a.view(np.uint8), b.view(np.uint8)) for a, b in zip(got, want)), prog.text
    assert seen > 0


@pytest.mark.parametrize("world", [1, 4, 8])
def test_reference_multinode_config_k32(world):
    """The reference's own two-node A100 machine (configs/a100_2node.json,
    axes [8,4], reduce {0}: K = 32 program devices, 254 programs) compiled
    for 32 slots on 1, 4 or 8 ranks: hazard-free plans equal to the oracle."""
    K, progs = golden_programs("a100_2node_r0")
    assert K == 32
    slot_rank = [d * world // K for d in range(K)]
    ctx = executor.Context.virtual(K, slot_rank, world)
    if world > 1:
        ctx.set_option("push_min_bytes", 0)
    for _, _, prog, _ in progs[::(1 if world == 1 else 5)]:
        desc = ctx.compile(prog, 1031, numeric.BF16).describe()
        inputs = numeric.synthetic_inputs(K, 1031, numeric.BF16)
        want = [x.copy() for x in inputs]
        numeric.execute(prog, K, want, numeric.BF16, nthreads=1)
        got = [x.copy() for x in inputs]
        simulate_plan(desc, got, numeric.BF16)
        assert all(np.array_equal(a.view(np.uint8), b.view(np.uint8)) for a, b in zip(got, want)), prog.text
