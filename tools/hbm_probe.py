#!/usr/bin/env python
"""HBM rates on this box for the mixes the local (1-GPU) steps issue:
read-only (sum), write-only (fill), copy (1 read + 1 write) and the step
kernel's own 1-read/3-write Broadcast over 8 x 256 MiB slots (local_ops.py
shape). CUDA events, best of --iters, buffers larger than L2.
  python tools/hbm_probe.py"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    import torch
    n = 1 << 30  # bf16 elements = 2 GiB
    x = torch.empty(n, dtype=torch.bfloat16, device="cuda").normal_()
    y = torch.empty_like(x)
    s = torch.cuda.current_stream()

    def best(fn, nbytes, iters=10):
        fn()
        torch.cuda.synchronize()
        out = 0.0
        for _ in range(iters):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(s)
            fn()
            b.record(s)
            torch.cuda.synchronize()
            out = max(out, nbytes / (a.elapsed_time(b) * 1e-3) / 1e9)
        return round(out, 1)

    import ctypes
    rt = None
    for name in ("libcudart.so", "libcudart.so.12"):
        try:
            rt = ctypes.CDLL(name)
            break
        except OSError:
            continue
    memset = None
    if rt is not None:
        rt.cudaMemsetAsync.argtypes = [ctypes.c_void_p, ctypes.c_int, ctypes.c_size_t, ctypes.c_void_p]
        memset = lambda: rt.cudaMemsetAsync(ctypes.c_void_p(y.data_ptr()), 0, 2 * n, ctypes.c_void_p(s.cuda_stream))
    res = {
        "read_only_sum_GBps": best(lambda: x.sum(dtype=torch.float32), 2 * n),
        "write_only_fill_GBps": best(lambda: y.fill_(1.0), 2 * n),
        "write_only_memset_GBps": best(memset, 2 * n) if memset else None,
        "copy_1r1w_GBps": best(lambda: y.copy_(x), 4 * n),
    }
    print(json.dumps(res), flush=True)


if __name__ == "__main__":
    main()
