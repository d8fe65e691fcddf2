"""Diagnostic: per-slot upload / run / download timings of the end-to-end
path (rs_ctx_upload, rs_plan_run, rs_ctx_download) on one GPU, to check
which stream each copy lands on. python tools/e2e_diag.py"""
import sys, time, torch
sys.path.insert(0, '.')
from paper_2110_10548_b200 import executor
K, ELEMS = 8, 128 << 20
ctx = executor.Context.local(K, [0]*K, 256 << 20)
host = {d: torch.empty(ELEMS, dtype=torch.bfloat16).pin_memory() for d in range(K)}
s = torch.cuda.current_stream()
for trial in range(3):
    torch.cuda.synchronize()
    a = torch.cuda.Event(enable_timing=True); b = torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter()
    a.record(s)
    for d in range(K): ctx.upload(d, host[d])
    b.record(s)
    torch.cuda.synchronize()
    print("upload 2GiB: events %.2f ms, wall %.2f ms" % (a.elapsed_time(b), (time.perf_counter()-t0)*1e3))
    a.record(s)
    for d in range(K): ctx.download(d, host[d])
    b.record(s)
    torch.cuda.synchronize()
    print("download 2GiB: events %.2f ms" % a.elapsed_time(b))
x = torch.empty(ELEMS*8, dtype=torch.bfloat16, device='cuda')
h = torch.empty(ELEMS*8, dtype=torch.bfloat16).pin_memory()
a.record(s); x.copy_(h, non_blocking=True); b.record(s); torch.cuda.synchronize()
print("torch H2D 2GiB %.2f ms" % a.elapsed_time(b))
