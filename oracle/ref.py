"""ctypes wrapper of the UNMODIFIED reference built by oracle/Makefile
(oracle/_ref/libredsynth_ref.so + oracle/ref_capi.cc).

TEST INFRASTRUCTURE ONLY. Exists only where /root/reference was present at
build time; callers must skip when `available()` is False.
"""
from __future__ import annotations

import ctypes
import json
import os

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB = os.path.join(HERE, "_ref", "libredsynth_ref.so")
_lib = None


def available() -> bool:
    return os.path.exists(LIB)


def lib():
    global _lib
    if _lib is None:
        _lib = ctypes.CDLL(LIB)
        PI = ctypes.POINTER(ctypes.c_int)
        _lib.ref_synthesize.argtypes = [ctypes.c_char_p, PI, ctypes.c_int, PI, ctypes.c_int, ctypes.c_int,
                                        ctypes.c_longlong, ctypes.c_int, ctypes.POINTER(ctypes.c_void_p)]
        _lib.ref_run_lowered.argtypes = [ctypes.c_int, PI, PI, PI, PI, ctypes.c_int,
                                         ctypes.POINTER(ctypes.c_ubyte), PI, PI, ctypes.c_void_p, ctypes.c_int]
        _lib.ref_time_run_lowered.argtypes = [ctypes.c_int, PI, PI, PI, PI, ctypes.c_int, ctypes.c_int]
        _lib.ref_time_run_lowered.restype = ctypes.c_double
        _lib.ref_report.argtypes = [ctypes.c_char_p, PI, ctypes.c_int, PI, ctypes.c_int, ctypes.c_int,
                                    ctypes.c_longlong, ctypes.c_int, ctypes.c_int,
                                    ctypes.POINTER(ctypes.c_void_p)]
        _lib.ref_free.argtypes = [ctypes.c_void_p]
    return _lib


def _ints(v):
    v = list(v)
    return (ctypes.c_int * max(1, len(v)))(*v)


def _take(ptr):
    try:
        return ctypes.string_at(ptr).decode()
    finally:
        lib().ref_free(ptr)


def synthesize(system_json: str, axes, reduce, size_limit=5, payload_bytes=1, algo=0):
    out = ctypes.c_void_p()
    rc = lib().ref_synthesize(system_json.encode(), _ints(axes), len(axes), _ints(reduce), len(reduce),
                              size_limit, payload_bytes, algo, ctypes.byref(out))
    text = _take(out)
    if rc != 0:
        raise RuntimeError(f"reference synthesize failed ({rc}): {text}")
    return json.loads(text)


def report(system_path: str, axes, reduce, payload_bytes, size_limit=5, algo=0, csv=False):
    out = ctypes.c_void_p()
    rc = lib().ref_report(system_path.encode(), _ints(axes), len(axes), _ints(reduce), len(reduce),
                          size_limit, payload_bytes, algo, 1 if csv else 0, ctypes.byref(out))
    text = _take(out)
    if rc != 0:
        raise RuntimeError(text)
    return text


def _csr(steps):
    ops = [op for op, _ in steps]
    sgp, gmp, mem = [0], [0], []
    for _, groups in steps:
        for g in groups:
            mem.extend(g)
            gmp.append(len(mem))
        sgp.append(len(gmp) - 1)
    return _ints(ops), _ints(sgp), _ints(gmp), _ints(mem)


def run_lowered(steps, k):
    """Reference RunLowered: returns (code, state bool[k,k,k] or None, step, violation, message)."""
    ops, sgp, gmp, mem = _csr(steps)
    state = (ctypes.c_ubyte * (k * k * k))()
    fs, fv = ctypes.c_int(-1), ctypes.c_int(0)
    msg = ctypes.create_string_buffer(512)
    rc = lib().ref_run_lowered(len(steps), ops, sgp, gmp, mem, k, state, ctypes.byref(fs), ctypes.byref(fv),
                               ctypes.addressof(msg), 512)
    st = np.frombuffer(bytes(state), dtype=np.uint8).reshape(k, k, k).astype(bool) if rc == 0 else None
    return rc, st, fs.value, fv.value, msg.value.decode()


def time_run_lowered(steps, k, iters=1000) -> float:
    ops, sgp, gmp, mem = _csr(steps)
    return lib().ref_time_run_lowered(len(steps), ops, sgp, gmp, mem, k, iters)
