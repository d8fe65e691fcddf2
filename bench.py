#!/usr/bin/env python
"""redsynth-b200 bench — BASELINE.json config 2 on B200.

Workload ("step"): execute EVERY synthesized program of config 2 once — all
placements of axes [2,4] on the [(node,1),(socket,2),(GPU,4)] descriptor,
reduce over axis 1 (254 programs) and over both axes (500 programs) — on
K = 8 program devices ("slots") holding 256 MiB of bf16 each (synthetic
N(0,1) data, rounded to bf16). With N GPUs the 8 slots are block-distributed
(N=1: all 8 slots in one GPU's HBM = "local reduction and copy"; N=8: one slot
per GPU, every step over NVLink/NVSwitch). Total work is fixed as N grows
("strong" scaling).

value = aggregate bus bandwidth of the step = sum over programs of
K * D * 2(n-1)/n (nccl-tests AllReduce bus bytes, n = reduction-group size,
D = 256 MiB) divided by the device-timed step (max over ranks).
e2e   = the same metric through the C-ABI from pinned HOST buffers: each
step uploads the 8 input buffers (rs_ctx_upload, 2 GiB), runs all programs
(rs_plan_run) and downloads the 8 results (rs_ctx_download, 2 GiB), all
inside the timed region.

Usage: python bench.py [--gpus N --steps K --warmup W] [--impl reference]
For N>1 launch under torchrun (one rank per GPU, NCCL process group).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = BASELINE_METRIC = "synthesized-program reduce time (µs) & speedup vs NCCL AllReduce; bus GB/s"
K_SLOTS = 8
D_BYTES = 256 << 20
DTYPE = "bf16"
ELEMS = D_BYTES // 2
REQUESTS = [[1], [0, 1]]
AXES = [2, 4]
SYSTEM = os.path.join(ROOT, "configs", "b200_sock.json")
# BASELINE.json configs 1-3: descriptor b200_sock
# [(node,1),(socket,2),(GPU,4)], 8 program devices ("slots").
WORKLOADS = {
    "config1": {"axes": [2, 4], "requests": [[0]], "bytes": 64 << 20, "dtype": "f32"},
    "config2": {"axes": [2, 4], "requests": [[1], [0, 1]], "bytes": 256 << 20, "dtype": "bf16"},
    "config3": {"axes": [2, 2, 2], "requests": [[0], [1], [2], [0, 1], [0, 2], [1, 2]], "bytes": 64 << 20,
                "dtype": "bf16"},
}
# --workload kN: K = N program devices, one per GPU (BASELINE config 4 descriptors)
K_DESCRIPTORS = {2: "b200_flat2", 4: "b200_sock4", 8: "b200_sock"}


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return float(p["hbm_gbs"]), "measured"
    except Exception:
        return 6650.0, "fallback"


NVLINK_PEAK_GBS = 770.0  # measured peer copy per direction (B200_PROFILING.md); nominal 900
HBM_NOMINAL_GBS = 7700.0  # HGX B200 HBM3e (B200_PROFILING.md); the roofline peak is the measured copy


def programs(axes=None, requests=None, payload=None, config=None):
    from paper_2110_10548_b200 import planner
    axes = AXES if axes is None else axes
    requests = REQUESTS if requests is None else requests
    payload = D_BYTES if payload is None else payload
    out = []
    for red in requests:
        syn = planner.synthesize(SYSTEM, axes, red, payload_bytes=payload)
        for mi, pl in enumerate(syn.placements):
            for pi, prog in enumerate(pl.programs):
                n = len(pl.partition[0])
                out.append({"request": red, "matrix": mi, "index": pi, "prog": prog, "group_size": n,
                            "factors": pl.factors, "partition": pl.partition, "config": config})
    return out


def bus_bytes(entry):
    n = entry["group_size"]
    return K_SLOTS * D_BYTES * 2.0 * (n - 1) / n


def algorithmic_link_bytes(prog, K, D):
    """per step, max over groups of f(op, n) * c_g with
    c_g = D * rows_g / K, rows_g = max non-empty rows over the members before
    or after the step (simulator.cc:156-182); f = 2(n-1)/n AllReduce,
    (n-1)/n ReduceScatter/AllGather, 1 Reduce/Broadcast."""
    import numpy as np
    from paper_2110_10548_b200 import planner
    f = {0: lambda n: 2 * (n - 1) / n, 1: lambda n: (n - 1) / n, 2: lambda n: (n - 1) / n,
         3: lambda n: 1.0, 4: lambda n: 1.0}
    total = 0.0
    prev = np.ones((K, K), dtype=bool)
    for s, (op, groups) in enumerate(prog.steps):
        post = planner.run_lowered(planner.LoweredProgram(steps=prog.steps[:s + 1]), K).any(axis=2)
        worst = 0.0
        for g in groups:
            rows = max(max(int(prev[d].sum()) for d in g), max(int(post[d].sum()) for d in g))
            worst = max(worst, f[op](len(g)) * D * rows / K)
        total += worst
        prev = post
    return total


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled during the timed region."""

    QUERY = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device_index):
        self.device_index = device_index
        self.proc = None
        self.lines = []
        self.thread = None

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={self.QUERY}", "--format=csv,noheader,nounits",
                                          "-i", str(self.device_index), "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._pump, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None

    def _pump(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.thread:
            self.thread.join(timeout=2)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in self.lines:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) < 9:
                continue
            try:
                sm.append(float(parts[1]))
                smax.append(float(parts[2]))
            except ValueError:
                continue
            for name, val in zip(names, parts[5:9]):
                if val.lower() == "active":
                    reasons.add(name)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def bench_config(workload, world, n_programs):
    """The `config` object of both arms (identical for the same workload)."""
    if workload == "config2":
        text = ("config 2: all 754 synthesized programs (axes [2,4] on b200_sock, reduce {1} "
                "and {0,1}), 8 slots x 256 MiB bf16")
    elif workload == "config3":
        text = (f"config 3: all {n_programs} synthesized programs (axes [2,2,2] on b200_sock, every single-axis "
                f"and two-axis request), 8 slots x 64 MiB bf16")
    else:
        text = (f"config 4 K={K_SLOTS}: all {n_programs} programs of {os.path.basename(SYSTEM)} axes {AXES}, "
                f"{K_SLOTS} slots x 256 MiB bf16")
    return {"workload": text, "slots_per_gpu": K_SLOTS // world, "programs": n_programs,
            "parallelism": f"{world} GPU(s), slots block-distributed",
            "l2": f"inputs larger than L2 (8 x {D_BYTES >> 20} MiB)"}


class _Prog:
    """A lowered program as the oracle reads it (steps of (op, groups))."""

    def __init__(self, doc):
        self.text = doc["text"]
        self.seconds = doc.get("seconds")
        self.steps = [(s["op"], [list(g) for g in s["groups"]]) for s in doc["steps"]]


def reference_programs():
    """The workload's program set from the REFERENCE itself: the unmodified
    reference library built by oracle/Makefile (oracle/_ref), else the golden
    fixtures it generated (tests/golden/programs_cfg2_*.json). Never from
    this repository's planner."""
    from oracle import ref
    out = []
    if ref.available():
        with open(SYSTEM) as f:
            system = f.read()
        docs = [ref.synthesize(system, AXES, red, payload_bytes=D_BYTES) for red in REQUESTS]
        source = "oracle/_ref (reference Synthesize)"
    else:
        names = {(1,): "cfg2_r1", (0, 1): "cfg2_r01"}
        docs = []
        for red in REQUESTS:
            with open(os.path.join(ROOT, "tests", "golden", f"programs_{names[tuple(red)]}.json")) as f:
                docs.append(json.load(f))
        source = "tests/golden (reference Synthesize fixtures)"
    for red, doc in zip(REQUESTS, docs):
        for mi, m in enumerate(doc["matrices"]):
            for pi, p in enumerate(m["programs"]):
                out.append({"request": red, "matrix": mi, "index": pi, "prog": _Prog(p),
                            "group_size": len(m["partition"][0])})
    return out, source


def run_reference(args):
    """--impl reference: the reference CPU path for this workload = the C
    numeric oracle (a restatement of semantics.cc:259-310 folded as
    dsl.cc:142-164; the reference's own RunLowered is symbolic and moves no
    data) on all host threads, over the reference's own program set. Each
    step executes one full-size program of the set (a spread over all 754,
    in order), so the run stays bounded. Touches nothing of this
    repository's package."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    if args.workload != "config2":
        print(json.dumps({"impl": "reference", "unavailable": "reference arm is defined for config2 only"}))
        return
    import numpy as np  # noqa: F401
    from oracle import numeric, ref
    progs, source = reference_programs()
    total = args.warmup + args.steps
    stride = max(1, len(progs) // max(1, total))
    order = [progs[(i * stride) % len(progs)] for i in range(total)]
    threads = numeric.hardware_threads()
    inputs = numeric.synthetic_inputs(K_SLOTS, ELEMS, numeric.BF16)
    times, bytes_ = [], []
    for it, e in enumerate(order):
        bufs = [x.copy() for x in inputs]
        t0 = time.perf_counter()
        numeric.execute(e["prog"], K_SLOTS, bufs, numeric.BF16, nthreads=threads)
        dt = time.perf_counter() - t0
        if it >= args.warmup:
            times.append(dt)
            bytes_.append(bus_bytes(e))
    value = sum(bytes_) / sum(times) / 1e9
    symbolic_us = None
    if ref.available():
        symbolic_us = statistics.mean(ref.time_run_lowered(e["prog"].steps, K_SLOTS, 2000) for e in order)
    sample = (f"{args.steps} timed programs (after {args.warmup} warm-up), one per step: every {stride}th of the "
              f"{len(progs)} programs from {source}, each at full size (8 x 256 MiB bf16)")
    line = {
        "impl": "reference", "metric": METRIC, "value": round(value, 3), "unit": "GB/s",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(1e3 * sum(times) / len(times), 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config("config2", args.gpus, len(progs)),
        "reference_sample": sample,
        "cpu_baseline": {"value": round(value, 3), "unit": "GB/s", "cores": threads, "cpu_model": cpu_model(),
                         "kind": "port", "sample": sample},
        "e2e": {"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "reference_runlowered_us_per_program": symbolic_us,
    }
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--e2e-serial", action="store_true", help="e2e without overlapping copies across steps")
    ap.add_argument("--no-graph", action="store_true", help="timed steps launch every program eagerly")
    ap.add_argument("--programs-out", default=None, help="write per-program device times (JSON)")
    ap.add_argument("--workload", default="config2", choices=["config2", "config3", "kN"],
                    help="config2: BASELINE config 2 (8 slots); config3: BASELINE config 3 (8 slots, 64 MiB); "
                         "kN: K = N slots, one per GPU")
    ap.add_argument("--no-rescore-all", action="store_true",
                    help="skip timing the programs of the other configs (1-3) for the simulator rescoring")
    ap.add_argument("--no-nvls", action="store_true", help="P2P kernels only (bit-exact everywhere)")
    ap.add_argument("--ranks-per-gpu", type=int, default=1,
                    help="(refused unless 1) ranks sharing a GPU spin on each other's flags from separate "
                         "launches, which B200 does not guarantee to co-schedule (Xid 109); the N=8 path is "
                         "exercised by emulated ranks in one cooperative launch instead "
                         "(tests/test_gpu_emulated_ranks.py)")
    ap.add_argument("--emulate-ranks", type=int, default=0,
                    help="dry run of the N-GPU plans on ONE GPU: N ranks emulated in one process "
                         "(rs_ctx_create_emulated, one cooperative launch per phase). Readiness of the N-rank "
                         "plans only (no IPC, NVLS or NCCL comparator); the times are not N-GPU numbers")
    ap.add_argument("--reduce-mode", type=int, default=None, help="executor Reduce variant (0 pull, 1 push, "
                    "2 NVLS, 3 NVLS root), for A/B runs")
    args = ap.parse_args()
    if args.impl == "reference":
        return run_reference(args)
    global K_SLOTS, SYSTEM, AXES, REQUESTS, D_BYTES, ELEMS, DTYPE
    if args.workload in WORKLOADS:
        wl = WORKLOADS[args.workload]
        AXES, REQUESTS, D_BYTES, DTYPE = wl["axes"], wl["requests"], wl["bytes"], wl["dtype"]
        ELEMS = D_BYTES // (2 if DTYPE == "bf16" else 4)
    if args.workload == "kN":
        from paper_2110_10548_b200 import planner as _pl
        K_SLOTS = args.gpus
        SYSTEM = _pl.config_path(K_DESCRIPTORS[args.gpus])
        AXES, REQUESTS = [args.gpus], [[0]]
    if not args.no_nvls:
        os.environ.setdefault("RS_NVLS", "1")  # used where a group has >= 4 slots on distinct GPUs

    import numpy as np
    import torch
    import torch.distributed as dist

    from paper_2110_10548_b200 import executor

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"--gpus {args.gpus} but WORLD_SIZE={world}")
    if args.ranks_per_gpu != 1:
        raise SystemExit("--ranks-per-gpu > 1 is refused: ranks that wait on each other must not share a GPU")
    rpg = 1
    device = local_rank // rpg
    torch.cuda.set_device(device)
    dev = torch.device("cuda", device)
    multi = world > 1
    if args.reduce_mode is not None:
        os.environ["RS_REDUCE_MODE"] = str(args.reduce_mode)
    if multi:
        if rpg > 1:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=dev)
    emu = args.emulate_ranks if not multi else 0
    pworld = emu or world  # ranks the plans are compiled for
    slot_rank = [d * pworld // K_SLOTS for d in range(K_SLOTS)]

    def make_ctx():
        if multi:
            return executor.Context.from_process_group(K_SLOTS, slot_rank, D_BYTES)
        if emu:
            return executor.Context.emulated(K_SLOTS, slot_rank, emu, device, D_BYTES)
        return executor.Context.local(K_SLOTS, [device] * K_SLOTS, D_BYTES)

    ctx = make_ctx()

    entries = programs(config=args.workload)
    # synthetic inputs for the slots this rank hosts (seed 1000+d)
    gen = torch.Generator(device=dev)
    for d in ctx.hosted_slots:
        gen.manual_seed(1000 + d)
        x = torch.randn(ELEMS, generator=gen, device=dev, dtype=torch.float32).to(torch.bfloat16)
        ctx.buffer(d, ELEMS, "bf16").copy_(x)
        del x
    torch.cuda.synchronize()
    plans = [ctx.compile(e["prog"], ELEMS, DTYPE) for e in entries]
    launches_per_step = sum(p.launches for p in plans)
    stream = torch.cuda.current_stream(dev)

    def barrier():
        if multi:
            dist.barrier()
        torch.cuda.synchronize()

    def step():
        for p in plans:
            p.run()

    for _ in range(args.warmup):
        step()
    barrier()
    ctx.synchronize()

    # per-program device times (outside the timed region): one untimed run
    # absorbs inter-rank skew, then two back-to-back runs are timed.
    prog_us = []
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in plans]
    for p, (a, b) in zip(plans, ev):
        p.run()
        a.record(stream)
        p.run()
        p.run()
        b.record(stream)
    barrier()
    prog_us = [a.elapsed_time(b) * 1e3 / 2 for a, b in ev]

    # NCCL's default AllReduce on the same bytes, one communicator per
    # reduction group (ReductionGroupPartition), all groups concurrently.
    nccl_us = {}
    comparator = None
    if multi and world == K_SLOTS:
        comparator = {"backend": "nccl" if rpg == 1 else "gloo (dry run: NCCL refuses two ranks on one GPU)",
                      "NCCL_NVLS_ENABLE": os.environ.get("NCCL_NVLS_ENABLE", "default"),
                      "NCCL_ALGO": os.environ.get("NCCL_ALGO", "default")}
        xbuf = torch.randn(ELEMS, device=dev).to(torch.bfloat16 if rpg == 1 else torch.float32)
        parts = {}
        for e in entries:
            parts.setdefault((tuple(e["request"]), e["matrix"]), e["partition"])
        for key, part in parts.items():
            groups = [dist.new_group(ranks=g) for g in part]
            mine = next(grp for grp, g in zip(groups, part) if rank in g)
            for _ in range(3):
                dist.all_reduce(xbuf, group=mine)
            barrier()
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(5):
                dist.all_reduce(xbuf, group=mine)
            b.record(stream)
            barrier()
            t = torch.tensor([a.elapsed_time(b) * 1e3 / 5], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            nccl_us[key] = float(t.item())
        del xbuf

    # The timed step replays one CUDA graph of all programs' launches (epochs
    # are device resident, so replays chain like eager runs); --no-graph
    # launches them one by one.
    graph = None
    if not args.no_graph:
        barrier()
        graph = torch.cuda.CUDAGraph()
        cap = torch.cuda.Stream(dev)
        cap.wait_stream(stream)
        with torch.cuda.stream(cap):
            with torch.cuda.graph(graph, stream=cap):
                step()
        barrier()
        graph.replay()  # one more warm-up step, through the graph
        barrier()

    sampler = ClockSampler(device) if rank == 0 else None
    if sampler:
        sampler.start()
    barrier()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    t0.record(stream)
    for _ in range(args.steps):
        if graph is not None:
            graph.replay()
        else:
            step()
    t1.record(stream)
    barrier()
    clocks = sampler.stop() if sampler else None
    ctx.synchronize()
    ms_local = t0.elapsed_time(t1)
    if multi:
        t = torch.tensor([ms_local], device=dev, dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_total = float(t.item())
        pu = torch.tensor(prog_us, device=dev, dtype=torch.float64)
        dist.all_reduce(pu, op=dist.ReduceOp.MAX)
        prog_us = pu.tolist()
    else:
        ms_total = ms_local
    ms_per_step = ms_total / args.steps
    bus_per_step = sum(bus_bytes(e) for e in entries)
    value = bus_per_step / (ms_per_step * 1e-3) / 1e9

    # roofline of the dominant (only) kernel: the step kernel
    if pworld == 1:
        alg = 0.0
        for p in plans:
            for s in range(p.program.num_steps):
                alg += p.step_bytes(s)[1]  # local mode: minimal HBM bytes of the tasks
        peak, peak_kind = load_peaks()
        achieved = alg / (ms_per_step * 1e-3) / 1e9
        traffic, tnote = None, "no ncu capture found"
        try:  # committed ncu --set full capture of the same kernel (profiles/)
            with open(os.path.join(ROOT, "profiles", "r02_ncu_local.json")) as f:
                cap = json.load(f)["launches"][0]
            traffic = cap["dram_bytes"]
            tnote = (f"traffic = dram read+write bytes of one profiled launch ({cap['what']}), "
                     f"{cap['dram_bytes'] / cap['algorithmic_bytes']:.3f} x its algorithmic bytes")
        except Exception:
            pass
        # The measured peak is torch's copy_ (1 read : 1 write); the step
        # kernel's 1:1 AllReduce launches run above it (ncu: 83 % of the DRAM
        # peak), so frac can exceed 1. The nominal 7.7 TB/s (B200_PROFILING.md)
        # is the physical ceiling and is reported beside it.
        roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                    "frac": round(achieved / peak, 4), "frac_of_nominal_7700": round(achieved / HBM_NOMINAL_GBS, 4),
                    "traffic": traffic,
                    "note": f"algorithmic bytes = sum over tasks of (sources + destinations) x range "
                            f"(minimal HBM traffic), per step {alg / 1e9:.2f} GB; peak {peak_kind} "
                            f"(torch copy_; frac > 1 = faster than that copy, the nominal 7.7 TB/s is the "
                            f"ceiling); {tnote}"}
    else:
        if pworld == K_SLOTS:
            alg = sum(algorithmic_link_bytes(e["prog"], K_SLOTS, D_BYTES) for e in entries)
        else:  # several slots per GPU: the plan's own per-GPU link bytes
            alg = sum(p.step_bytes(s)[0] for p in plans for s in range(p.program.num_steps))
        achieved = alg / (ms_per_step * 1e-3) / 1e9
        traffic, tnote = None, "no NVLink capture found"
        try:  # committed ncu capture of the cross-GPU kernel (tools/profile_p2p.py, profiles/)
            with open(os.path.join(ROOT, "profiles", "r01_ncu_nvlink.json")) as f:
                caps = json.load(f)
            cap = caps.get(f"k{min(pworld, 4)}_push") or next(iter(caps.values()))  # large steps push
            traffic = cap["nvlrx_user"] + cap["nvltx_user"]
            tnote = (f"traffic = NVLink user bytes rx+tx of one profiled launch ({cap['what']}, replayed alone), "
                     f"{traffic / cap['own_share_algorithmic']:.4f} x its algorithmic bytes; link headers and flags "
                     f"on top: tx +{cap['nvltx_total'] / cap['nvltx_user'] - 1:.0%} (profiles/r01_ncu_nvlink.txt)")
        except Exception:
            pass
        roofline = {"bound": "nvlink", "achieved": round(achieved, 1), "peak": NVLINK_PEAK_GBS, "unit": "GB/s",
                    "frac": round(achieved / NVLINK_PEAK_GBS, 4), "frac_of_nominal_900": round(achieved / 900.0, 4),
                    "traffic": traffic,
                    "note": "per-GPU per-direction link bytes of SURVEY §8(d) (T_roof = sum_s max_g f*c_g) "
                            "over the measured step; peak = measured peer copy 770 GB/s (900 nominal); " + tnote}

    # per (request, placement): baseline AllReduce and best synthesized program
    instances = {}
    for e, us in zip(entries, prog_us):
        key = (tuple(e["request"]), e["matrix"])
        inst = instances.setdefault(key, {"request": e["request"], "factors": e["factors"], "best_us": 1e30,
                                          "best": None, "allreduce_us": None, "programs": 0})
        inst["programs"] += 1
        if e["index"] == 0:
            inst["allreduce_us"] = round(us, 2)
        if us < inst["best_us"]:
            inst["best_us"], inst["best"] = round(us, 2), e["prog"].text
    for key, inst in instances.items():
        if key in nccl_us:
            inst["nccl_allreduce_us"] = round(nccl_us[key], 2)
            inst["speedup_vs_nccl"] = round(nccl_us[key] / inst["best_us"], 4)
    inst_list = list(instances.values())
    speedups = [i["speedup_vs_nccl"] for i in inst_list if "speedup_vs_nccl" in i]
    speedup_vs_nccl = round(float(statistics.geometric_mean(speedups)), 4) if speedups else None
    from paper_2110_10548_b200 import rescore
    # Config 5 rows (reference Simulate vs measured, and the B200-calibrated
    # model rs_plan_predict_us: per launch, measured latency + the plan's own
    # link / HBM bytes at the measured rates; local launches ~3 us,
    # cross-GPU ~8 us incl. handshake). Configs other than this workload's are
    # timed at the end (outside every timed region) and added.
    cal_args = dict(launch_us=3.0, link_gbs=650.0, hbm_gbs=5967.0) if pworld == 1 else \
        dict(launch_us=8.0, link_gbs=650.0, hbm_gbs=5967.0)
    resc_rows = [{"instance": (args.workload, tuple(e["request"]), e["matrix"]), "index": e["index"],
                  "sim_seconds": e["prog"].seconds, "cal_us": p.predict_us(**cal_args), "measured_us": us,
                  "text": e["prog"].text} for e, p, us in zip(entries, plans, prog_us)]

    # End to end through the C-ABI from pinned HOST memory: every step
    # uploads the hosted slots' inputs (rs_ctx_upload), runs the step's
    # programs (rs_plan_run), and downloads the results (rs_ctx_download).
    # Pipelined across steps with two buffer sets (two contexts, A/B): the
    # upload of step i+1 and the download of step i-1 overlap step i's
    # programs on their own copy streams (PCIe is full duplex); the timed
    # region spans the first upload to the last download.
    e2e = None
    if not args.no_e2e:
        host_in = {d: ctx.buffer(d, ELEMS, "bf16").cpu().pin_memory() for d in ctx.hosted_slots}
        e2e_steps = max(2, min(args.steps, 8))  # the first upload and last download are not overlapped
        sets = [(ctx, plans)]
        if not args.e2e_serial:
            ctx_b = make_ctx()
            sets.append((ctx_b, [ctx_b.compile(e["prog"], ELEMS, DTYPE) for e in entries]))
            for p in sets[1][1]:  # warm the second set (untimed)
                p.run()
        host_out = [{d: torch.empty_like(t).pin_memory() for d, t in host_in.items()} for _ in sets]
        # the programs of each buffer set as one CUDA graph (as in the timed step)
        set_graphs = []
        for _, ps in sets:
            if args.no_graph:
                set_graphs.append(None)
                continue
            barrier()
            g = torch.cuda.CUDAGraph()
            cap = torch.cuda.Stream(dev)
            cap.wait_stream(stream)
            with torch.cuda.stream(cap):
                with torch.cuda.graph(g, stream=cap):
                    for p in ps:
                        p.run()
            barrier()
            set_graphs.append(g)
        h2d = torch.cuda.Stream(dev)
        d2h = torch.cuda.Stream(dev)
        h2d_h, d2h_h = executor._stream_handle(h2d), executor._stream_handle(d2h)
        barrier()
        h0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        h2d.wait_event(e0)
        freed = [None] * len(sets)
        for i in range(e2e_steps):
            x = i % len(sets)
            c, ps = sets[x]
            if freed[x] is not None:  # results of this set's previous step are out
                h2d.wait_event(freed[x])
            for d, t in host_in.items():
                c.upload(d, t, stream=h2d_h)
            up = torch.cuda.Event()
            up.record(h2d)
            stream.wait_event(up)
            if set_graphs[x] is not None:
                set_graphs[x].replay()
            else:
                for p in ps:
                    p.run()
            done = torch.cuda.Event()
            done.record(stream)
            d2h.wait_event(done)
            for d, t in host_out[x].items():
                c.download(d, t, stream=d2h_h)
            freed[x] = torch.cuda.Event()
            freed[x].record(d2h)
        for ev_ in freed:
            if ev_ is not None:
                stream.wait_event(ev_)
        e1.record(stream)
        barrier()
        e2e_ms = e0.elapsed_time(e1) / e2e_steps
        if multi:
            t = torch.tensor([e2e_ms], device=dev, dtype=torch.float64)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_ms = float(t.item())
        wall_ms = (time.perf_counter() - h0) * 1e3 / e2e_steps
        nbytes = K_SLOTS * D_BYTES
        e2e = {"value": round(bus_per_step / (e2e_ms * 1e-3) / 1e9, 3),
               "unit": "GB/s", "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes,
               "sample": f"{e2e_steps} steps ({len(plans)} programs each), each between an H2D of the {K_SLOTS} "
                         f"input buffers and a D2H of its results, pinned host memory; "
                         + ("serial" if len(sets) == 1 else
                            "pipelined over two buffer sets (copies of neighbouring steps overlap compute)"),
               "ms_per_step": round(e2e_ms, 2), "wall_ms_per_step": round(wall_ms, 2)}
        del set_graphs
        if len(sets) > 1:
            barrier()
            for p in sets[1][1]:
                p.close()
            sets[1][0].close()
        del host_in, host_out

    cpu = None
    if rank == 0 and pworld == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(entries, args.workload)

    # Config 5 over configs 1-3 (BASELINE.json): time every program of the
    # other configs (one warm run, then two back-to-back runs per program,
    # max over ranks) in a 64 MiB context, outside every timed region.
    rescore_configs = [args.workload] if args.workload in WORKLOADS else []
    if args.workload in WORKLOADS and not args.no_rescore_all:
        barrier()
        if multi:
            extra_ctx = executor.Context.from_process_group(K_SLOTS, slot_rank, 64 << 20)
        elif emu:
            extra_ctx = executor.Context.emulated(K_SLOTS, slot_rank, emu, device, 64 << 20)
        else:
            extra_ctx = executor.Context.local(K_SLOTS, [device] * K_SLOTS, 64 << 20)
        for name in ("config1", "config2", "config3"):
            wl = WORKLOADS[name]
            if name == args.workload or wl["bytes"] > (64 << 20):
                continue
            es = 2 if wl["dtype"] == "bf16" else 4
            ents = programs(wl["axes"], wl["requests"], wl["bytes"], config=name)
            ps = [extra_ctx.compile(e["prog"], wl["bytes"] // es, wl["dtype"]) for e in ents]
            evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in ps]
            barrier()
            for p, (a, b) in zip(ps, evs):
                p.run()
                a.record(stream)
                p.run()
                p.run()
                b.record(stream)
            barrier()
            us = [a.elapsed_time(b) * 1e3 / 2 for a, b in evs]
            if multi:
                t = torch.tensor(us, device=dev, dtype=torch.float64)
                dist.all_reduce(t, op=dist.ReduceOp.MAX)
                us = t.tolist()
            resc_rows += [{"instance": (name, tuple(e["request"]), e["matrix"]), "index": e["index"],
                           "sim_seconds": e["prog"].seconds, "cal_us": p.predict_us(**cal_args), "measured_us": u,
                           "text": e["prog"].text} for e, p, u in zip(ents, ps, us)]
            for p in ps:
                p.close()
            rescore_configs.append(name)
        barrier()
        extra_ctx.close()

    def topk_block(key, extra):
        res = rescore.topk([dict(r, sim_seconds=r[key]) for r in resc_rows])
        by_cfg = {}
        for c in rescore_configs:
            sub = rescore.topk([dict(r, sim_seconds=r[key]) for r in resc_rows if r["instance"][0] == c])
            by_cfg[c] = {"instances": sub["instances"], "top_k": sub["top_k"],
                         "top_k_tie_aware": sub["top_k_tie_aware"], "spearman": sub["spearman"]}
        out = {"instances": res["instances"], "configs": rescore_configs, "top_k": res["top_k"],
               "top_k_tie_aware": res["top_k_tie_aware"], "spearman": res["spearman"], "by_config": by_cfg}
        out.update(extra)
        return out

    sim_topk = topk_block("sim_seconds", {"model": "reference Simulate (ring, b200_sock bandwidths)"})
    cal_topk = topk_block("cal_us", {"model": cal_args})

    if args.programs_out and rank == 0:
        with open(args.programs_out, "w") as f:
            json.dump([{"config": r["instance"][0], "request": list(r["instance"][1]), "matrix": r["instance"][2],
                        "index": r["index"], "text": r["text"], "sim_seconds": r["sim_seconds"],
                        "calibrated_us": r["cal_us"], "measured_us": r["measured_us"]} for r in resc_rows], f)

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(ms_per_step, 3), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": bench_config(args.workload, pworld, len(entries)),
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": launches_per_step * args.steps,
            "clocks": clocks,
            "program_us": {"mean": round(statistics.mean(prog_us), 2), "min": round(min(prog_us), 2),
                           "max": round(max(prog_us), 2)},
            "instances": inst_list,
            "simulator_rescoring": sim_topk,
            "calibrated_rescoring": cal_topk,
            "speedup_vs_nccl": speedup_vs_nccl,
            "comparator": comparator,
            "nvls": bool(getattr(ctx, "nvls", False)) if world > 1 else False,
            "scaling_note": ("strong scaling of a fixed 8-slot workload: at N=1 every collective is an HBM-local "
                             "sum/copy (no NVLink), at N=2/4 several slots share a GPU and every step crosses "
                             "NVLink, at N=8 one slot per GPU; value is a nccl-tests-style bus figure, so the N=1 "
                             "number measures HBM, the N>1 numbers NVLink"),
        }
        if emu:
            line["dry_run"] = (f"{emu} ranks emulated on one GPU (own heaps, one cooperative launch per phase): "
                               f"readiness of the N={emu} plans only (no IPC, NVLS or NCCL comparator); times are "
                               f"not {emu}-GPU numbers")
            line["emulated_ranks"] = emu
        print(json.dumps(line), flush=True)
    barrier()
    for p in plans:
        p.close()
    if multi:
        dist.barrier()
    ctx.close()
    if multi:
        dist.destroy_process_group()


def cpu_baseline(entries, workload="config2"):
    """The C oracle on this host's cores over a bounded sample (2 programs
    of config 2 at full size), reported beside the GPU number."""
    try:
        from oracle import numeric
    except Exception as exc:  # pragma: no cover
        return {"value": None, "unavailable": str(exc)}
    threads = numeric.hardware_threads()
    inputs = numeric.synthetic_inputs(K_SLOTS, ELEMS, numeric.BF16)
    # Programs spread over the whole set, run until ~10 s of CPU time.
    order = [entries[(i * 97) % len(entries)] for i in range(len(entries))]
    t = 0.0
    b = 0.0
    done = 0
    while t < 10.0 and done < len(order):
        e = order[done]
        bufs = [x.copy() for x in inputs]
        t0 = time.perf_counter()
        numeric.execute(e["prog"], K_SLOTS, bufs, numeric.BF16, nthreads=threads)
        t += time.perf_counter() - t0
        b += bus_bytes(e)
        done += 1
    return {"value": round(b / t / 1e9, 3), "unit": "GB/s", "cores": threads, "cpu_model": cpu_model(),
            "kind": "port",
            "sample": f"{done} {workload} programs (every 97th of the {len(entries)}, in order) at full size "
                      f"({K_SLOTS} x {D_BYTES >> 20} MiB bf16), ~10 s of CPU time",
            "seconds": round(t, 2)}


if __name__ == "__main__":
    main()
