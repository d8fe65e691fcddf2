"""Pins the C numeric oracle (oracle/numeric.c) before anything is checked
against it:
  * boolean layer == the reference RunLowered (golden program sets reach the
    goal partition; the 300 golden refusals give the same code/step/violation);
  * int32: every program ends with device i = sum of its reduction group's
    inputs (exact, order-free identity — independent of any implementation);
  * f32 / bf16 / i32: identical to an independent pure-numpy restatement of
    semantics.cc:259-310 written here, and to the committed golden vectors.
"""
import json
import os

import numpy as np
import pytest

from common import GOLDEN, bf16_round, bf16_widen, golden_programs
from oracle import numeric


def _goal_held(K, partition):
    held = np.zeros((K, K), dtype=np.uint64)
    for grp in partition:
        mask = 0
        for d in grp:
            mask |= 1 << d
        for d in grp:
            held[d, :] = mask
    return held


@pytest.mark.parametrize("name", ["cfg1", "cfg2_r1", "cfg2_r01", "cfg3_r01", "cfg3_r12", "k8_sock"])
def test_boolean_layer_reaches_reference_goal(name):
    K, progs = golden_programs(name)
    for _, _, prog, part in progs:
        assert (numeric.check(prog, K) == _goal_held(K, part)).all(), prog.text


def test_boolean_layer_refusals_match_reference():
    from paper_2110_10548_b200.planner import LoweredProgram
    cases = json.load(open(os.path.join(GOLDEN, "refusals.json")))
    for c in cases:
        prog = LoweredProgram(steps=[(op, gs) for op, gs in c["steps"]])
        if c["code"] == 0:
            held = numeric.check(prog, 8)
            assert held.astype(int).tolist() == c["held"]
        else:
            with pytest.raises(numeric.OracleViolation) as e:
                numeric.check(prog, 8)
            assert (e.value.code, e.value.step, e.value.violation) == (c["code"], c["step"], c["violation"])


@pytest.mark.parametrize("name,N", [("cfg1", 1000), ("cfg2_r1", 997), ("cfg2_r01", 64), ("cfg3_r02", 21),
                                    ("k8_sock", 5), ("a100_2node_r0", 100)])
def test_int32_group_sum_identity(name, N):
    K, progs = golden_programs(name)
    inputs = numeric.synthetic_inputs(K, N, numeric.I32)
    for _, _, prog, part in progs:
        bufs = [x.copy() for x in inputs]
        numeric.execute(prog, K, bufs, numeric.I32, nthreads=1)
        for grp in part:
            expect = sum(inputs[d].astype(np.int64) for d in grp).astype(np.int32)
            for d in grp:
                assert np.array_equal(bufs[d], expect), (prog.text, d)


# ---- independent restatement (pure numpy) of the data semantics ------------

def _restated(prog, K, bufs, dtype):
    """Literal per-group fold of semantics.cc:259-310 over the row chunking."""
    N = bufs[0].size
    lo = [r * N // K for r in range(K + 1)]
    held = [[1 << d] * K for d in range(K)]  # column masks per (device,row)

    def ssum(srcs):
        if dtype == numeric.F32:
            acc = srcs[0].copy()
            for x in srcs[1:]:
                acc = (acc + x).astype(np.float32)
            return acc
        if dtype == numeric.BF16:
            acc = bf16_widen(srcs[0])
            for x in srcs[1:]:
                acc = (acc + bf16_widen(x)).astype(np.float32)
            return bf16_round(acc)
        acc = srcs[0].copy()
        for x in srcs[1:]:
            acc = (acc + x).astype(np.int32)
        return acc

    for op, groups in prog.steps:
        for g in groups:
            rows = [r for r in range(K) if held[g[0]][r]]
            if op in (0, 3):  # AllReduce / Reduce
                for r in rows:
                    s = ssum([bufs[m][lo[r]:lo[r + 1]] for m in g])
                    for m in (g if op == 0 else g[:1]):
                        bufs[m][lo[r]:lo[r + 1]] = s
                uni = [0] * K
                for r in range(K):
                    for m in g:
                        uni[r] |= held[m][r]
                for m in g:
                    held[m] = list(uni) if (op == 0 or m == g[0]) else [0] * K
            elif op == 1:  # ReduceScatter
                run = len(rows) // len(g)
                uni = [0] * K
                for r in range(K):
                    for m in g:
                        uni[r] |= held[m][r]
                for i, r in enumerate(rows):
                    owner = g[i // run]
                    bufs[owner][lo[r]:lo[r + 1]] = ssum([bufs[m][lo[r]:lo[r + 1]] for m in g])
                for mi, m in enumerate(g):
                    held[m] = [uni[r] if (r in rows[mi * run:(mi + 1) * run]) else 0 for r in range(K)]
            elif op == 2:  # AllGather
                uni = [0] * K
                for r in range(K):
                    for m in g:
                        if held[m][r]:
                            for o in g:
                                if o != m:
                                    bufs[o][lo[r]:lo[r + 1]] = bufs[m][lo[r]:lo[r + 1]]
                        uni[r] |= held[m][r]
                for m in g:
                    held[m] = list(uni)
            else:  # Broadcast
                for r in range(K):
                    if held[g[0]][r]:
                        for m in g[1:]:
                            bufs[m][lo[r]:lo[r + 1]] = bufs[g[0]][lo[r]:lo[r + 1]]
                for m in g[1:]:
                    held[m] = list(held[g[0]])


@pytest.mark.parametrize("dtype", [numeric.F32, numeric.BF16, numeric.I32])
@pytest.mark.parametrize("name,N", [("cfg1", 203), ("cfg3_r01", 45), ("cfg2_r1", 17)])
def test_oracle_equals_independent_restatement(name, N, dtype):
    K, progs = golden_programs(name)
    inputs = numeric.synthetic_inputs(K, N, dtype)
    for _, _, prog, _ in progs[:120]:
        a = [x.copy() for x in inputs]
        b = [x.copy() for x in inputs]
        numeric.execute(prog, K, a, dtype, nthreads=1)
        _restated(prog, K, b, dtype)
        for d in range(K):
            assert np.array_equal(a[d].view(np.uint8), b[d].view(np.uint8)), (prog.text, d)


def test_oracle_matches_committed_vectors():
    doc = json.load(open(os.path.join(GOLDEN, "numeric_small.json")))
    K, N = doc["K"], doc["N"]
    cfg1 = golden_programs("cfg1")[1]
    by = {(mi, pi): prog for mi, pi, prog, _ in cfg1}
    for v in doc["vectors"]:
        bufs = numeric.synthetic_inputs(K, N, v["dtype"])
        numeric.execute(by[(v["matrix"], v["program"])], K, bufs, v["dtype"], nthreads=1)
        view = np.uint32 if v["dtype"] == numeric.F32 else None
        got = [(b.view(view) if view else b).tolist() for b in bufs]
        assert got == v["out"]


def test_multithreaded_equals_single_threaded():
    K, progs = golden_programs("cfg2_r01")
    inputs = numeric.synthetic_inputs(K, 1 << 18, numeric.BF16)
    for _, _, prog, _ in progs[::50]:
        a = [x.copy() for x in inputs]
        b = [x.copy() for x in inputs]
        numeric.execute(prog, K, a, numeric.BF16, nthreads=1)
        numeric.execute(prog, K, b, numeric.BF16, nthreads=8)
        assert all(np.array_equal(x, y) for x, y in zip(a, b))


@pytest.mark.parametrize("N", [0, 1, 3, 7, 8, 9])
def test_tiny_and_ragged_buffers(N):
    """N < K leaves some rows empty (zero elements); the int32 identity holds."""
    K, progs = golden_programs("cfg2_r01")
    inputs = numeric.synthetic_inputs(K, N, numeric.I32)
    for _, _, prog, part in progs[::25]:
        bufs = [x.copy() for x in inputs]
        numeric.execute(prog, K, bufs, numeric.I32, nthreads=1)
        for grp in part:
            expect = sum(inputs[d].astype(np.int64) for d in grp).astype(np.int32)
            assert all(np.array_equal(bufs[d], expect) for d in grp)
