#!/usr/bin/env python
"""NVLink traffic counters through NVML (no profiler): validates the units of
the NVML field values against a known peer copy, so bench.py can report the
measured link bytes of a timed region next to the algorithmic ones.

  python tools/nvlink_counters.py          # needs >= 2 GPUs

Prints, per field and scope, the counter delta for a D-byte copy GPU0 -> GPU1.
"""
from __future__ import annotations

import ctypes
import sys

import pynvml

FIELDS = ["NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX",
          "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_TX", "NVML_FI_DEV_NVLINK_THROUGHPUT_RAW_RX",
          "NVML_FI_DEV_NVLINK_COUNT_XMIT_BYTES", "NVML_FI_DEV_NVLINK_COUNT_RCV_BYTES"]
ALL_LINKS = 0xFFFFFFFF


def value(v):
    t = v.valueType
    u = v.value
    return {0: u.dVal, 1: u.uiVal, 2: u.ulVal, 3: u.ullVal, 4: u.sllVal, 5: u.siVal}.get(t, u.ullVal)


def read(h, nlinks):
    out = {}
    for name in FIELDS:
        fid = getattr(pynvml, name, None)
        if fid is None:
            continue
        for scope in [ALL_LINKS] + list(range(nlinks)):
            try:
                v = pynvml.nvmlDeviceGetFieldValues(h, [(fid, scope)])[0]
            except pynvml.NVMLError:
                continue
            if v.nvmlReturn != 0:
                continue
            out[(name, scope)] = value(v)
    return out


def gpm_sample(h):
    smp = pynvml.nvmlGpmSampleAlloc()
    pynvml.nvmlGpmSampleGet(h, smp)
    return smp


def gpm_rates(s1, s2):
    """NVLink total TX/RX rates between two GPM samples (NVML reports MiB/s)."""
    mg = pynvml.c_nvmlGpmMetricsGet_t()
    mg.version = pynvml.NVML_GPM_METRICS_GET_VERSION
    mg.numMetrics = 2
    mg.sample1 = s1
    mg.sample2 = s2
    mg.metrics[0].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_TX_PER_SEC
    mg.metrics[1].metricId = pynvml.NVML_GPM_METRIC_NVLINK_TOTAL_RX_PER_SEC
    pynvml.nvmlGpmMetricsGet(mg)
    return [(mg.metrics[i].nvmlReturn, mg.metrics[i].value) for i in range(2)]


def main():
    import time
    import torch
    pynvml.nvmlInit()
    hs = [pynvml.nvmlDeviceGetHandleByIndex(i) for i in range(2)]
    nlinks = 18
    D = 1 << 30
    a = torch.empty(D, dtype=torch.uint8, device="cuda:0")
    b = torch.empty(D, dtype=torch.uint8, device="cuda:1")
    b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    for h in hs:
        try:
            sup = pynvml.nvmlGpmQueryDeviceSupport(h)
            print("GPM supported:", sup.isSupportedDevice)
        except pynvml.NVMLError as e:
            print("GPM query failed:", e)
    for name in FIELDS:
        fid = getattr(pynvml, name, None)
        try:
            v = pynvml.nvmlDeviceGetFieldValues(hs[0], [(fid, ALL_LINKS), (fid, 0)])
            print(name, "ret", v[0].nvmlReturn, v[1].nvmlReturn)
        except pynvml.NVMLError as e:
            print(name, "error", e)
    before = [read(h, nlinks) for h in hs]
    try:
        g1 = [gpm_sample(h) for h in hs]
    except pynvml.NVMLError as e:
        g1 = None
        print("GPM sample failed:", e)
    t0 = time.perf_counter()
    reps = 4
    for _ in range(reps):
        b.copy_(a)
    torch.cuda.synchronize(0)
    torch.cuda.synchronize(1)
    dt = time.perf_counter() - t0
    after = [read(h, nlinks) for h in hs]
    if g1 is not None:
        g2 = [gpm_sample(h) for h in hs]
        for g in range(2):
            r = gpm_rates(g1[g], g2[g])
            print(f"gpu{g} GPM nvlink tx/rx (ret, value): {r}; x interval {dt:.4f}s -> "
                  f"tx {r[0][1] * dt * 2**20 / (reps * D):.4f} x bytes (if MiB/s), "
                  f"{r[0][1] * dt * 1e6 / (reps * D):.4f} x bytes (if MB/s)")
    print(f"copy GPU0 -> GPU1, {reps} x {D} bytes = {reps * D / 2**30:.1f} GiB")
    for g in range(2):
        for key in sorted(after[g], key=lambda k: (k[0], k[1])):
            d = after[g][key] - before[g].get(key, 0)
            if key[1] == ALL_LINKS or d:
                scope = "all" if key[1] == ALL_LINKS else f"link{key[1]}"
                print(f"gpu{g} {key[0]:45s} {scope:6s} delta {d}  (= {d / (reps * D):.4f} x bytes, "
                      f"{d * 1024 / (reps * D):.4f} x KiB-units)")
    return 0


if __name__ == "__main__":
    sys.exit(main())
