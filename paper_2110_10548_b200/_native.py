"""ctypes binding of libredsynth_b200.so (include/redsynth_exec.h).

The shared library is built in-tree by ``make`` (or ``__graft_entry__.build()``)
into ``paper_2110_10548_b200/_lib/``. There is no fallback: if the library is
missing, every entry point raises ``NativeLibraryMissing``.
"""
from __future__ import annotations

import ctypes
import os
import threading

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_DIR = os.path.join(_HERE, "_lib")
LIB_PATH = os.environ.get("RS_LIB_PATH") or os.path.join(LIB_DIR, "libredsynth_b200.so")

RS_OK = 0
RS_INVALID_ARGUMENT = 3
RS_FAILED_PRECONDITION = 9
RS_INTERNAL = 13
RS_UNAVAILABLE = 14

RS_F32, RS_BF16, RS_I32 = 0, 1, 2
RS_MAX_RANKS = 8
RS_IPC_HANDLE_BYTES = 64

# Every symbol include/redsynth_exec.h declares (checked by the CPU tests).
EXPORTED_SYMBOLS = (
    "rs_last_error", "rs_version",
    "rs_ctx_create", "rs_ctx_create_rank", "rs_ctx_ipc_handle", "rs_ctx_open_peers", "rs_ctx_create_emulated",
    "rs_ctx_create_virtual", "rs_plan_describe_json", "rs_ctx_set_option", "rs_ctx_nvls",
    "rs_ctx_set_exchange", "rs_ctx_upload", "rs_ctx_download",
    "rs_ctx_destroy", "rs_ctx_buffer", "rs_ctx_local_ranks", "rs_ctx_synchronize",
    "rs_plan_compile", "rs_plan_run", "rs_plan_run_host", "rs_plan_launch_count",
    "rs_plan_step_bytes", "rs_plan_predict_us", "rs_plan_set_launch", "rs_plan_set_option", "rs_plan_destroy", "rs_plan_time",
    "rs_synthesize_json", "rs_report", "rs_run_lowered", "rs_free",
)


class NativeLibraryMissing(RuntimeError):
    pass


class ExecError(RuntimeError):
    """A non-OK status from the executor; ``code`` mirrors absl::StatusCode."""

    def __init__(self, code: int, message: str):
        super().__init__(f"[{_CODE_NAMES.get(code, code)}] {message}")
        self.code = code
        self.message = message


_CODE_NAMES = {3: "INVALID_ARGUMENT", 9: "FAILED_PRECONDITION", 13: "INTERNAL", 14: "UNAVAILABLE"}

_lib = None
_lock = threading.Lock()

_P = ctypes.c_void_p
_I = ctypes.c_int
_PI = ctypes.POINTER(ctypes.c_int)
_PI32 = ctypes.POINTER(ctypes.c_int32)
_SZ = ctypes.c_size_t
# int (*)(const void* send, size_t bytes, void* recv, void* user)
EXCHANGE_FN = ctypes.CFUNCTYPE(ctypes.c_int, ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)


def _declare(lib):
    sig = {
        "rs_last_error": (ctypes.c_char_p, []),
        "rs_version": (ctypes.c_char_p, []),
        "rs_ctx_create": (_I, [_I, _PI, _SZ, ctypes.POINTER(_P)]),
        "rs_ctx_create_rank": (_I, [_I, _PI, _I, _I, _I, _SZ, ctypes.POINTER(_P)]),
        "rs_ctx_ipc_handle": (_I, [_P, _P]),
        "rs_ctx_create_virtual": (_I, [_I, _PI, _I, ctypes.POINTER(_P)]),
        "rs_ctx_create_emulated": (_I, [_I, _PI, _I, _I, _SZ, ctypes.POINTER(_P)]),
        "rs_plan_describe_json": (_I, [_P, ctypes.POINTER(ctypes.c_void_p)]),
        "rs_ctx_set_option": (_I, [_P, ctypes.c_char_p, ctypes.c_longlong]),
        "rs_ctx_nvls": (_I, [_P, _PI]),
        "rs_ctx_upload": (_I, [_P, _I, _P, _SZ, _P]),
        "rs_ctx_download": (_I, [_P, _I, _P, _SZ, _P]),
        "rs_ctx_set_exchange": (_I, [_P, EXCHANGE_FN, _P]),
        "rs_ctx_open_peers": (_I, [_P, _P]),
        "rs_ctx_destroy": (_I, [_P]),
        "rs_ctx_buffer": (_I, [_P, _I, ctypes.POINTER(_P)]),
        "rs_ctx_local_ranks": (_I, [_P, _PI, _PI]),
        "rs_ctx_synchronize": (_I, [_P]),
        "rs_plan_compile": (_I, [_P, _I, _PI32, _PI32, _PI32, _PI32, _SZ, _I, ctypes.POINTER(_P)]),
        "rs_plan_run": (_I, [_P, _P, _P]),
        "rs_plan_run_host": (_I, [_P, _P, _P]),
        "rs_plan_launch_count": (_I, [_P, _PI]),
        "rs_plan_step_bytes": (_I, [_P, _I, ctypes.POINTER(ctypes.c_double), ctypes.POINTER(ctypes.c_double)]),
        "rs_plan_predict_us": (_I, [_P, ctypes.c_double, ctypes.c_double, ctypes.c_double,
                                    ctypes.POINTER(ctypes.c_double)]),
        "rs_plan_set_launch": (_I, [_P, _I, _I]),
        "rs_plan_set_option": (_I, [_P, ctypes.c_char_p, ctypes.c_longlong]),
        "rs_plan_destroy": (_I, [_P]),
        "rs_plan_time": (_I, [_P, _I, _I, ctypes.POINTER(ctypes.c_double)]),
        "rs_synthesize_json": (_I, [ctypes.c_char_p, _PI, _I, _PI, _I, _I, ctypes.c_longlong, _I,
                                    ctypes.POINTER(ctypes.c_void_p)]),
        "rs_report": (_I, [ctypes.c_char_p, _PI, _I, _PI, _I, _I, ctypes.c_longlong, _I, _I,
                           ctypes.POINTER(ctypes.c_void_p)]),
        "rs_run_lowered": (_I, [_I, _PI32, _PI32, _PI32, _PI32, _I, ctypes.POINTER(ctypes.c_ubyte), _PI, _PI]),
        "rs_free": (None, [ctypes.c_void_p]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args


def lib():
    """The loaded library (raises NativeLibraryMissing, never falls back)."""
    global _lib
    with _lock:
        if _lib is None:
            if not os.path.exists(LIB_PATH):
                raise NativeLibraryMissing(
                    f"{LIB_PATH} is missing: build it with `make` or __graft_entry__.build(); "
                    "the executor has no CPU fallback")
            handle = ctypes.CDLL(LIB_PATH, mode=ctypes.RTLD_GLOBAL)
            _declare(handle)
            _lib = handle
    return _lib


def check(code: int) -> None:
    if code != RS_OK:
        msg = lib().rs_last_error().decode(errors="replace")
        raise ExecError(code, msg)


def take_string(ptr: ctypes.c_void_p) -> str:
    """Copies a malloc'ed C string returned by the library and frees it."""
    try:
        return ctypes.string_at(ptr).decode()
    finally:
        lib().rs_free(ptr)


def int_array(values, ctype=ctypes.c_int):
    values = list(values)
    return (ctype * max(1, len(values)))(*values)
