"""Python mirror of the host planner (C++ in csrc/planner, API of
/root/reference/proj/include/redsynth/*.h), reached through the C-ABI.

``synthesize`` = EnumerateMatrices + Synthesize (+ Simulate) for every
placement (reference report.cc:132-208 without the ranking), ``report`` =
RunPipeline + ReportToJson/Csv (byte-identical to the reference tool), and
``run_lowered`` = the reference's symbolic executor RunLowered (dsl.cc:142).
"""
from __future__ import annotations

import ctypes
import json
import os
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as nat

COLLECTIVES = ("AllReduce", "ReduceScatter", "AllGather", "Reduce", "Broadcast")
OP = {name: i for i, name in enumerate(COLLECTIVES)}
VIOLATIONS = ("none", "group has fewer than two devices", "device outside the state context",
              "devices hold different chunk sets", "chunk already reduced on another device",
              "chunk count not divisible by group size", "gather sources hold overlapping chunk sets",
              "broadcast root lacks data held by a member", "broadcast would not add information")

_CONFIG_DIR = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "configs")


def config_path(name: str) -> str:
    """Path of a shipped machine config (configs/<name>.json)."""
    return os.path.join(_CONFIG_DIR, name if name.endswith(".json") else name + ".json")


@dataclass
class LoweredProgram:
    """Steps of (collective index, groups of physical device ids) — the
    reference's LoweredProgram (dsl.h:74-79) as plain Python data."""

    steps: list = field(default_factory=list)  # [(op:int, [[int,...],...]), ...]
    text: str = ""
    seconds: float | None = None  # reference cost-model prediction, if known

    def to_csr(self):
        ops = np.array([op for op, _ in self.steps], dtype=np.int32)
        sgp = [0]
        gmp = [0]
        members = []
        for _, groups in self.steps:
            for g in groups:
                members.extend(g)
                gmp.append(len(members))
            sgp.append(len(gmp) - 1)
        return (ops, np.array(sgp, dtype=np.int32), np.array(gmp, dtype=np.int32),
                np.array(members if members else [0], dtype=np.int32))

    @property
    def num_steps(self) -> int:
        return len(self.steps)

    def max_group_size(self) -> int:
        return max((len(g) for _, gs in self.steps for g in gs), default=1)

    @staticmethod
    def from_json(entry) -> "LoweredProgram":
        return LoweredProgram(steps=[(s["op"], [list(g) for g in s["groups"]]) for s in entry["steps"]],
                              text=entry.get("text", ""), seconds=entry.get("seconds"))


@dataclass
class Placement:
    factors: list
    partition: list
    hierarchy: list
    programs: list  # [LoweredProgram], emission order

    def baseline_index(self) -> int:
        """Index of `Slice(root) InsideGroup AllReduce` (report.cc:35-46)."""
        for i, p in enumerate(self.programs):
            if p.text == "Slice(root) InsideGroup AllReduce":
                return i
        return -1


@dataclass
class Synthesis:
    device_count: int
    placements: list  # [Placement]


def _system_text(system) -> str:
    if isinstance(system, dict):
        return json.dumps(system)
    if isinstance(system, str) and system.lstrip().startswith("{"):
        return system
    path = system if os.path.exists(system) else config_path(system)
    with open(path) as f:
        return f.read()


def synthesize(system, axes: Sequence[int], reduce: Sequence[int], *, size_limit: int = 5,
               payload_bytes: int = 1, algo: str = "ring") -> Synthesis:
    lib = nat.lib()
    out = ctypes.c_void_p()
    nat.check(lib.rs_synthesize_json(_system_text(system).encode(), nat.int_array(axes), len(axes),
                                     nat.int_array(reduce), len(reduce), size_limit,
                                     int(payload_bytes), 1 if algo == "tree" else 0, ctypes.byref(out)))
    doc = json.loads(nat.take_string(out))
    placements = [Placement(factors=m["factors"], partition=m["partition"], hierarchy=m["hierarchy"],
                            programs=[LoweredProgram.from_json(p) for p in m["programs"]])
                  for m in doc["matrices"]]
    return Synthesis(device_count=doc["device_count"], placements=placements)


def report(system_path: str, axes, reduce, payload_bytes: int, *, size_limit: int = 5,
           algo: str = "ring", fmt: str = "json") -> str:
    lib = nat.lib()
    out = ctypes.c_void_p()
    nat.check(lib.rs_report(system_path.encode(), nat.int_array(axes), len(axes), nat.int_array(reduce),
                            len(reduce), size_limit, int(payload_bytes), 1 if algo == "tree" else 0,
                            1 if fmt == "csv" else 0, ctypes.byref(out)))
    return nat.take_string(out)


class RuleViolationError(nat.ExecError):
    def __init__(self, code, message, step, violation):
        super().__init__(code, message)
        self.step = step
        self.violation = violation


def run_lowered(program: LoweredProgram, k: int) -> np.ndarray:
    """Symbolic execution; returns bool[k, k, k] (device, row, column)."""
    lib = nat.lib()
    ops, sgp, gmp, mem = program.to_csr()
    state = np.zeros(k * k * k, dtype=np.uint8)
    fs, fv = ctypes.c_int(-1), ctypes.c_int(0)
    p32 = ctypes.POINTER(ctypes.c_int32)
    code = lib.rs_run_lowered(len(program.steps), ops.ctypes.data_as(p32), sgp.ctypes.data_as(p32),
                              gmp.ctypes.data_as(p32), mem.ctypes.data_as(p32), k,
                              state.ctypes.data_as(ctypes.POINTER(ctypes.c_ubyte)), ctypes.byref(fs),
                              ctypes.byref(fv))
    if code != 0:
        raise RuleViolationError(code, lib.rs_last_error().decode(), fs.value, fv.value)
    return state.reshape(k, k, k).astype(bool)
