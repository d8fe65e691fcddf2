"""Shared helpers for the test-suite (loads golden program sets, builds the
numpy plan simulator used by the CPU plan-compiler tests)."""
import json
import os

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")

GOLDEN_SETS = ["cfg1", "cfg2_r1", "cfg2_r01", "cfg3_r0", "cfg3_r1", "cfg3_r2", "cfg3_r01", "cfg3_r02",
               "cfg3_r12", "k2_flat", "k4_flat", "k4_sock", "k8_flat", "k8_sock", "a100_2node_r0"]


def load_golden(name):
    with open(os.path.join(GOLDEN, f"programs_{name}.json")) as f:
        return json.load(f)


def golden_programs(name):
    """[(matrix index, program index, LoweredProgram, partition)]"""
    from paper_2110_10548_b200.planner import LoweredProgram
    doc = load_golden(name)
    out = []
    for mi, m in enumerate(doc["matrices"]):
        for pi, p in enumerate(m["programs"]):
            out.append((mi, pi, LoweredProgram.from_json(p), m["partition"]))
    return doc["device_count"], out


def bf16_round(x_f32):
    import ml_dtypes
    return x_f32.astype(ml_dtypes.bfloat16).view(np.uint16)


def bf16_widen(u16):
    return (u16.astype(np.uint32) << 16).view(np.float32)


LL_REGION = -3


def simulate_plan(desc, bufs, dtype):
    """Executes a compiled plan (Plan.describe()) over numpy slot buffers.

    Every task of a step is checked for hazards first (a byte written by one
    task may not be touched by another task of the same step), then executed:
    dst_j = src_0 + src_1 + ... in source order (f32 adds / bf16 via f32 with
    one RNE rounding / wrapping i32), a single source being a raw copy —
    exactly the step kernel's contract. Returns nothing; bufs are updated."""
    es = 2 if dtype == 1 else 4
    view = {0: np.float32, 1: np.uint16, 2: np.int32}[dtype]
    scratch = {}

    def mem(slot, region):
        if region < 0:
            return bufs[slot]
        key = (slot, region)
        if key not in scratch:  # fresh scratch holds garbage: poison it
            scratch[key] = np.full(bufs[slot].nbytes, 0x5A, dtype=np.uint8).view(bufs[slot].dtype)
        return scratch[key]

    for step in desc["steps"]:
        for rank, r in enumerate(step["ranks"]):
            for t in r["tasks"]:
                t["rank"] = rank
        every = [t for r in step["ranks"] for t in r["tasks"]]
        # Push variant: landing tasks (mode 3) complete a chunk before the
        # reducing tasks (mode 4) read it (chunk flags), so they form a
        # sub-phase of their own; everything else runs after them.
        for tasks in ([t for t in every if t.get("mode") == 3], [t for t in every if t.get("mode") != 3]):
            _simulate_tasks(tasks, every, bufs, mem, scratch, es, view, dtype)


def _simulate_tasks(tasks, every, bufs, mem, scratch, es, view, dtype):
    if True:
        for t in tasks:
            t.setdefault("src_region", [-1] * len(t["src"]))
            t.setdefault("dst_region", [-1] * len(t["dst"]))
        # One-shot (LL) sources (region -3) are packets of the source slot that
        # some task on the source's GPU read and sent to this task's GPU.
        for t in tasks:
            for s, rg in zip(t["src"], t["src_region"]):
                if rg != LL_REGION:
                    continue
                assert any(u["mode"] == 2 and (s, -1) in zip(u["src"], u["src_region"]) and
                           (u["lo"], u["hi"]) == (t["lo"], t["hi"]) and t["rank"] in u["sends"]
                           for u in every), f"no sender for LL source {s} of {t}"
        # hazard check: per memory object, written intervals vs every other task's accesses
        acc = {}
        for i, t in enumerate(tasks):
            for s, rg in zip(t["src"], t["src_region"]):
                if rg == LL_REGION:
                    continue
                acc.setdefault((s, rg), []).append((t["lo"], t["hi"], i, "r"))
            for d, rg in zip(t["dst"], t["dst_region"]):
                acc.setdefault((d, rg), []).append((t["lo"], t["hi"], i, "w"))
        for slot, ivs in acc.items():
            ivs.sort()
            for a in range(len(ivs)):
                for b in range(a + 1, len(ivs)):
                    if ivs[b][0] >= ivs[a][1]:
                        break
                    if ivs[a][2] != ivs[b][2] and "w" in (ivs[a][3], ivs[b][3]):
                        raise AssertionError(f"hazard on slot {slot}: {ivs[a]} vs {ivs[b]}")
        snap = {k: v.copy() for k, v in bufs.items()} if isinstance(bufs, dict) else [b.copy() for b in bufs]
        snap_scratch = {k: v.copy() for k, v in scratch.items()}

        def src_mem(slot, region):
            if region in (-1, LL_REGION):
                return snap[slot]
            if (slot, region) in snap_scratch:
                return snap_scratch[(slot, region)]
            return mem(slot, region)

        for t in tasks:
            assert t["lo"] % es == 0 and t["hi"] % es == 0
            if t.get("mode") == 2:
                if not t["dst"]:
                    continue
            elif t["vec"]:  # (push landing / reducing bodies are 16-byte aligned too)
                assert t["lo"] % 16 == 0 and t["hi"] % 16 == 0
            else:
                assert t["hi"] - t["lo"] < 32
            lo, hi = t["lo"] // es, t["hi"] // es
            srcs = [src_mem(s, rg).view(view)[lo:hi] for s, rg in zip(t["src"], t["src_region"])]
            if len(srcs) == 1:
                out = srcs[0].copy()
            elif dtype == 0:
                out = srcs[0].copy()
                for x in srcs[1:]:
                    out = (out + x).astype(np.float32)
            elif dtype == 1:
                accf = bf16_widen(srcs[0])
                for x in srcs[1:]:
                    accf = (accf + bf16_widen(x)).astype(np.float32)
                out = bf16_round(accf)
            else:
                out = srcs[0].copy()
                for x in srcs[1:]:
                    out = (out + x).astype(np.int32)
            for d, rg in zip(t["dst"], t["dst_region"]):
                mem(d, rg).view(view)[lo:hi] = out
