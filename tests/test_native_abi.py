"""The C-ABI library loads on a CPU-only machine and exports every symbol
include/redsynth_exec.h declares; calls that need a GPU fail with a status
code instead of crashing. No compute is attempted here."""
import ctypes
import os
import re

import pytest

from common import ROOT
from paper_2110_10548_b200 import _native as nat


def _declared():
    text = open(os.path.join(ROOT, "include", "redsynth_exec.h")).read()
    return sorted(set(re.findall(r"\b(rs_[a-z_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert sorted(nat.EXPORTED_SYMBOLS) == _declared()


def test_library_exports_every_declared_symbol():
    lib = nat.lib()
    for name in _declared():
        assert hasattr(lib, name), name
    assert b"sm_100a" in lib.rs_version()


def test_sass_is_sm100a():
    # the executor library carries an sm_100a cubin (cuobjdump lists the arch)
    import shutil
    import subprocess
    exe = shutil.which("cuobjdump") or "/usr/local/cuda/bin/cuobjdump"
    if not os.path.exists(exe):
        pytest.skip("cuobjdump not available")
    out = subprocess.run([exe, "--list-elf", nat.LIB_PATH], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_create_without_gpu_reports_status():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    h = ctypes.c_void_p()
    code = nat.lib().rs_ctx_create(2, nat.int_array([0, 0]), 1 << 20, ctypes.byref(h))
    assert code in (nat.RS_UNAVAILABLE, nat.RS_INTERNAL, nat.RS_INVALID_ARGUMENT)
    assert nat.lib().rs_last_error()


def test_null_arguments_are_invalid():
    lib = nat.lib()
    assert lib.rs_ctx_create(2, None, 1 << 20, None) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_plan_run(None, None, None) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_ctx_destroy(None) == nat.RS_OK


def test_option_and_model_errors_on_a_planning_context():
    """Options and the cost model on a planning-only (virtual) context: bad
    keys / values are INVALID_ARGUMENT with a message naming the valid keys;
    runs are refused (no GPU work is attempted)."""
    from paper_2110_10548_b200 import executor
    from paper_2110_10548_b200.planner import LoweredProgram
    ctx = executor.Context.virtual(4, [0, 1, 2, 3], 4)
    lib = nat.lib()
    assert lib.rs_ctx_set_option(ctx._h, b"no_such_option", 1) == nat.RS_INVALID_ARGUMENT
    assert b"ll_max_bytes" in lib.rs_last_error()
    for key in (b"push_min_bytes", b"ll_max_bytes", b"nvls_min_bytes", b"barrier_timeout_ms"):
        assert lib.rs_ctx_set_option(ctx._h, key, 1 << 20) == nat.RS_OK
    plan = ctx.compile(LoweredProgram(steps=[(0, [[0, 1, 2, 3]])]), 1024, "f32")
    us = ctypes.c_double()
    assert lib.rs_plan_predict_us(plan._h, 8.0, -1.0, 6000.0, ctypes.byref(us)) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_plan_predict_us(plan._h, 8.0, 650.0, 6000.0, None) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_plan_predict_us(plan._h, 8.0, 650.0, 6000.0, ctypes.byref(us)) == nat.RS_OK and us.value > 8.0
    assert lib.rs_plan_run(plan._h, None, None) == nat.RS_FAILED_PRECONDITION
    assert b"virtual" in lib.rs_last_error()
    plan.close()
    ctx.close()


def test_emulated_context_argument_checks():
    """rs_ctx_create_emulated validates its arguments before touching a GPU
    (world in [2, RS_MAX_RANKS], slot ranks in range) and reports a status
    without a GPU."""
    lib = nat.lib()
    h = ctypes.c_void_p()
    assert lib.rs_ctx_create_emulated(4, None, 2, 0, 1 << 20, ctypes.byref(h)) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_ctx_create_emulated(4, nat.int_array([0, 0, 1, 1]), 1, 0, 1 << 20,
                                      ctypes.byref(h)) == nat.RS_INVALID_ARGUMENT
    assert b"world_size" in lib.rs_last_error()
    assert lib.rs_ctx_create_emulated(4, nat.int_array([0, 0, 1, 1]), 9, 0, 1 << 20,
                                      ctypes.byref(h)) == nat.RS_INVALID_ARGUMENT
    import torch
    if not torch.cuda.is_available():
        code = lib.rs_ctx_create_emulated(4, nat.int_array([0, 0, 1, 1]), 2, 0, 1 << 20, ctypes.byref(h))
        assert code in (nat.RS_UNAVAILABLE, nat.RS_INTERNAL, nat.RS_INVALID_ARGUMENT)


def test_plan_options_validated():
    """Named plan knobs (unroll, threads, max_ctas, wide_loads, dynamic_pieces,
    pdl, local_wide, vec256, remote256, piece_queue) are accepted; unknown keys and bad
    values are INVALID_ARGUMENT naming the valid keys."""
    from paper_2110_10548_b200 import executor
    from paper_2110_10548_b200.planner import LoweredProgram
    ctx = executor.Context.virtual(4, [0, 1, 2, 3], 4)
    plan = ctx.compile(LoweredProgram(steps=[(0, [[0, 1, 2, 3]])]), 1024, "f32")
    lib = nat.lib()
    for key, val in ((b"unroll", 8), (b"threads", 256), (b"max_ctas", 0), (b"wide_loads", 0), (b"dynamic_pieces", 1),
                     (b"pdl", 0), (b"local_wide", 0), (b"vec256", 2), (b"remote256", 1),
                     (b"piece_queue", 2), (b"push_prefetch", 0)):
        assert lib.rs_plan_set_option(plan._h, key, val) == nat.RS_OK, key
    assert lib.rs_plan_set_option(plan._h, b"unroll", 3) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_plan_set_option(plan._h, b"piece_queue", 3) == nat.RS_INVALID_ARGUMENT
    assert lib.rs_plan_set_option(plan._h, b"piece_queue", -1) == nat.RS_OK
    assert lib.rs_plan_set_option(plan._h, b"bogus", 1) == nat.RS_INVALID_ARGUMENT
    assert b"piece_queue" in lib.rs_last_error()
    for key in (b"ll_total_bytes", b"reduce_push_min_bytes", b"reduce_wave_bytes", b"push_wave_bytes"):
        assert lib.rs_ctx_set_option(ctx._h, key, 1 << 20) == nat.RS_OK, key
    assert lib.rs_ctx_set_option(ctx._h, b"wave_lag", 2) == nat.RS_OK
    assert lib.rs_ctx_set_option(ctx._h, b"wave_lag", -1) == nat.RS_INVALID_ARGUMENT
    plan.close()
    ctx.close()
