"""The checked build (make checked: device-side assertions on task ranges,
piece ownership, and the epoch protocol — no one-shot packet and no push
chunk flag from a later epoch) run on the driver's box: local mode and
emulated ranks (world 4 and 8, every cross-rank variant, graph replays),
in a subprocess so that the release library of this session stays loaded.
Any assertion raises the rank's error flag (code >= 2), which
rs_ctx_synchronize reports — the subprocess then fails."""
import os
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("no CUDA device", allow_module_level=True)

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CHECKED = os.path.join(ROOT, "paper_2110_10548_b200", "_lib", "libredsynth_b200_checked.so")

SCRIPT = r"""
import os, sys
sys.path.insert(0, {root!r}); sys.path.insert(0, {tests!r})
import numpy as np
from common import golden_programs
from oracle import numeric
from paper_2110_10548_b200 import _native, executor
assert _native.LIB_PATH.endswith("libredsynth_b200_checked.so"), _native.LIB_PATH
import test_gpu_emulated_ranks as T
import ranks_worker
# local mode: every config-2 program, bf16
ctx = executor.Context.local(8, [0] * 8, 1 << 20)
K, progs = golden_programs("cfg2_r01")
inputs = numeric.synthetic_inputs(K, 3001, numeric.BF16)
for _, _, prog, _ in progs:
    for d in range(K):
        ctx.write(d, inputs[d])
    plan = ctx.compile(prog, 3001, "bf16"); plan.run(); ctx.synchronize()
    want = [x.copy() for x in inputs]; numeric.execute(prog, K, want, numeric.BF16)
    assert all(np.array_equal(ctx.read(d, 6002), want[d].view(np.uint8)) for d in range(K)), prog.text
    plan.close()
ctx.close()
# emulated ranks: every variant with graph replays
for world in (4, 8):
    ctxs, used = {{}}, {{}}
    for case in ranks_worker.default_cases(world):
        T._run_case(ctxs, world, case, used)
    for c in ctxs.values():
        c.close()
    assert all(used.get(v, 0) > 0 for v in ("ll", "pull", "push", "reduce_push")), used
print("CHECKED_OK")
"""


def test_checked_build_local_and_emulated_ranks():
    if not os.path.exists(CHECKED):
        pytest.skip("checked build missing (make checked)")
    env = dict(os.environ, RS_LIB_PATH=CHECKED, RS_BARRIER_TIMEOUT_S="20")
    r = subprocess.run([sys.executable, "-c", SCRIPT.format(root=ROOT, tests=HERE)], env=env, cwd=HERE,
                       capture_output=True, text=True, timeout=1200)
    assert r.returncode == 0 and "CHECKED_OK" in r.stdout, r.stdout[-3000:] + r.stderr[-3000:]
