"""ctypes wrapper of oracle/_ref/liboracle_numeric.so (oracle/numeric.c).

TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "liboracle_numeric.so")
F32, BF16, I32 = 0, 1, 2
_lib = None


class OracleViolation(RuntimeError):
    def __init__(self, code, step, violation):
        super().__init__(f"oracle refused program: code {code}, step {step}, violation {violation}")
        self.code, self.step, self.violation = code, step, violation


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB):
            subprocess.check_call(["make", "-s", "-C", HERE, "numeric"])
        _lib = ctypes.CDLL(LIB)
        p32 = ctypes.POINTER(ctypes.c_int32)
        _lib.oracle_execute.argtypes = [ctypes.c_int, ctypes.c_int, p32, p32, p32, p32, ctypes.c_size_t,
                                        ctypes.c_int, ctypes.POINTER(ctypes.c_void_p), ctypes.c_int,
                                        ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                        ctypes.POINTER(ctypes.c_uint64)]
        _lib.oracle_check.argtypes = [ctypes.c_int, ctypes.c_int, p32, p32, p32, p32,
                                      ctypes.POINTER(ctypes.c_int), ctypes.POINTER(ctypes.c_int),
                                      ctypes.POINTER(ctypes.c_uint64)]
        _lib.oracle_hardware_threads.restype = ctypes.c_int
    return _lib


def hardware_threads() -> int:
    return lib().oracle_hardware_threads()


def _csr(program):
    ops = np.array([op for op, _ in program.steps], dtype=np.int32)
    sgp, gmp, mem = [0], [0], []
    for _, groups in program.steps:
        for g in groups:
            mem.extend(g)
            gmp.append(len(mem))
        sgp.append(len(gmp) - 1)
    return (ops if len(ops) else np.zeros(1, np.int32), np.array(sgp, np.int32), np.array(gmp, np.int32),
            np.array(mem or [0], np.int32))


def execute(program, K: int, bufs, dtype: int, nthreads: int = 0):
    """Runs `program` in place over K numpy buffers (f32 / uint16-as-bf16 /
    int32). Returns the final held-row masks uint64[K, K]."""
    ops, sgp, gmp, mem = _csr(program)
    elems = bufs[0].size
    ptrs = (ctypes.c_void_p * K)(*[ctypes.c_void_p(b.ctypes.data) for b in bufs])
    held = np.zeros(K * K, dtype=np.uint64)
    fs, fv = ctypes.c_int(-1), ctypes.c_int(0)
    p32 = ctypes.POINTER(ctypes.c_int32)
    rc = lib().oracle_execute(K, len(program.steps), ops.ctypes.data_as(p32), sgp.ctypes.data_as(p32),
                              gmp.ctypes.data_as(p32), mem.ctypes.data_as(p32), elems, dtype, ptrs,
                              nthreads, ctypes.byref(fs), ctypes.byref(fv),
                              held.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    if rc != 0:
        raise OracleViolation(rc, fs.value, fv.value)
    return held.reshape(K, K)


def check(program, K: int):
    ops, sgp, gmp, mem = _csr(program)
    held = np.zeros(K * K, dtype=np.uint64)
    fs, fv = ctypes.c_int(-1), ctypes.c_int(0)
    p32 = ctypes.POINTER(ctypes.c_int32)
    rc = lib().oracle_check(K, len(program.steps), ops.ctypes.data_as(p32), sgp.ctypes.data_as(p32),
                            gmp.ctypes.data_as(p32), mem.ctypes.data_as(p32), ctypes.byref(fs),
                            ctypes.byref(fv), held.ctypes.data_as(ctypes.POINTER(ctypes.c_uint64)))
    if rc != 0:
        raise OracleViolation(rc, fs.value, fv.value)
    return held.reshape(K, K)


def synthetic_inputs(K: int, elems: int, dtype: int, seed_base: int = 1000):
    """SURVEY.md §8(d) inputs: seed 1000+d; int32 uniform [-2^20, 2^20);
    f32 standard normal; bf16 = RNE(f32) stored as uint16."""
    out = []
    for d in range(K):
        rng = np.random.default_rng(seed_base + d)
        if dtype == I32:
            out.append(rng.integers(-(1 << 20), 1 << 20, size=elems, dtype=np.int32))
        else:
            x = rng.standard_normal(elems, dtype=np.float32)
            if dtype == F32:
                out.append(x)
            else:
                import ml_dtypes
                out.append(x.astype(ml_dtypes.bfloat16).view(np.uint16))
    return out
