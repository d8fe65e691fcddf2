"""Diagnostic: NVLS bf16 AllReduce on 2 GPUs against the single-rounded
ordered sum, printing the elements that differ (the switch's bf16 reduction
is not correctly rounded; profiles/r01_nvls_bf16_n2_rounding.txt)."""
import os, sys, numpy as np
sys.path.insert(0, os.getcwd()); sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
os.environ["RS_NVLS"] = "1"
import torch
from common import golden_programs, bf16_widen
from oracle import numeric
from paper_2110_10548_b200 import executor
ctx = executor.Context.local(2, [0, 1], max_bytes=64 << 20)
print("nvls", ctx.nvls)
ctx.set_option("nvls_min_group", 2); ctx.set_option("nvls_min_bytes", 0); ctx.set_option("ll_max_bytes", 0)
K, progs = golden_programs("k2_flat")
prog = progs[0][2]
for N in (4099, 1 << 20):
    inputs = numeric.synthetic_inputs(K, N, numeric.BF16)
    for d in range(K): ctx.write(d, inputs[d])
    plan = ctx.compile(prog, N, "bf16")
    print(N, [t.get("mode") for st in plan.describe()["steps"] for rk in st["ranks"] for t in rk["tasks"]][:8])
    plan.run(); ctx.synchronize()
    y = bf16_widen(ctx.read(0, N * 2).view(np.uint16)).astype(np.float64)
    x0 = bf16_widen(inputs[0].view(np.uint16)).astype(np.float64); x1 = bf16_widen(inputs[1].view(np.uint16)).astype(np.float64)
    ex = x0 + x1
    # reference: single RNE rounding of exact sum
    want = numeric.synthetic_inputs(K, N, numeric.BF16); numeric.execute(prog, K, want, numeric.BF16)
    w = bf16_widen(want[0].view(np.uint16)).astype(np.float64)
    diff = np.nonzero(y != w)[0]
    print("N", N, "mismatch vs single-rounding", len(diff))
    for i in diff[:12]:
        print(i, x0[i], x1[i], "exact", ex[i], "got", y[i], "want", w[i])
    plan.close()
ctx.close()
