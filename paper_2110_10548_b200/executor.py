"""Python host mirror of the B200 executor (C-ABI: include/redsynth_exec.h).

Reference interface it sits next to: ``RunLowered(const LoweredProgram&, int k,
StepFailure*)`` (/root/reference/proj/include/redsynth/dsl.h:108). Same program
input, same refusal behaviour (FAILED_PRECONDITION naming the step and the
violated rule), but it moves real data: every step becomes one hand-written
sm_100a kernel per GPU over NVSwitch peer memory.

Two ways to build a context:
  * ``Context.local(K, ordinals)`` — one process drives every GPU (slots may
    share a GPU; K slots on one GPU = HBM-local mode);
  * ``Context.from_process_group(K, slot_rank)`` — one process per GPU under
    torch.distributed; IPC handles are exchanged with all_gather_object.
PyTorch is used only for plumbing (streams, tensors aliasing the slot
buffers through DLPack, the process group). There is no CPU fallback: a
missing library raises.
"""
from __future__ import annotations

import ctypes
from typing import Optional, Sequence

import numpy as np

from . import _native as nat
from .planner import LoweredProgram

DTYPES = {"f32": nat.RS_F32, "float32": nat.RS_F32, "bf16": nat.RS_BF16, "bfloat16": nat.RS_BF16,
          "i32": nat.RS_I32, "int32": nat.RS_I32}
ELEM_BYTES = {nat.RS_F32: 4, nat.RS_BF16: 2, nat.RS_I32: 4}


def dtype_code(dtype) -> int:
    if isinstance(dtype, int):
        return dtype
    name = str(dtype).replace("torch.", "")
    return DTYPES[name]


# ---- DLPack view of a raw device pointer (zero-copy torch tensor) ----------

class _DLDevice(ctypes.Structure):
    _fields_ = [("device_type", ctypes.c_int32), ("device_id", ctypes.c_int32)]


class _DLDataType(ctypes.Structure):
    _fields_ = [("code", ctypes.c_uint8), ("bits", ctypes.c_uint8), ("lanes", ctypes.c_uint16)]


class _DLTensor(ctypes.Structure):
    _fields_ = [("data", ctypes.c_void_p), ("device", _DLDevice), ("ndim", ctypes.c_int32),
                ("dtype", _DLDataType), ("shape", ctypes.POINTER(ctypes.c_int64)),
                ("strides", ctypes.POINTER(ctypes.c_int64)), ("byte_offset", ctypes.c_uint64)]


class _DLManagedTensor(ctypes.Structure):
    pass


_DELETER = ctypes.CFUNCTYPE(None, ctypes.POINTER(_DLManagedTensor))
_DLManagedTensor._fields_ = [("dl_tensor", _DLTensor), ("manager_ctx", ctypes.c_void_p),
                             ("deleter", _DELETER)]
_KEEP = {}


@_DELETER
def _dl_deleter(ptr):
    _KEEP.pop(ctypes.addressof(ptr.contents), None)


def device_tensor(ptr: int, numel: int, dtype_name: str, device_id: int):
    """torch tensor aliasing `numel` elements at device pointer `ptr`."""
    import torch
    code, bits = {"f32": (2, 32), "bf16": (4, 16), "i32": (0, 32), "u8": (1, 8)}[dtype_name]
    shape = (ctypes.c_int64 * 1)(numel)
    mt = _DLManagedTensor()
    mt.dl_tensor = _DLTensor(ctypes.c_void_p(ptr), _DLDevice(2, device_id), 1, _DLDataType(code, bits, 1),
                             shape, None, 0)
    mt.deleter = _dl_deleter
    _KEEP[ctypes.addressof(mt)] = (mt, shape)
    pycapsule_new = ctypes.pythonapi.PyCapsule_New
    pycapsule_new.restype = ctypes.py_object
    pycapsule_new.argtypes = [ctypes.c_void_p, ctypes.c_char_p, ctypes.c_void_p]
    capsule = pycapsule_new(ctypes.addressof(mt), b"dltensor", None)
    return torch.utils.dlpack.from_dlpack(capsule)


# ---- context / plan ---------------------------------------------------------

_CUDA_STREAM_LEGACY = 0x1  # cudaStreamLegacy


def _stream_handle(stream) -> int:
    """torch stream -> cudaStream_t for the C-ABI. torch's default stream is
    the legacy NULL stream; pass it explicitly as cudaStreamLegacy because the
    C-ABI reads NULL as "the context's own stream"."""
    h = stream.cuda_stream
    return h if h else _CUDA_STREAM_LEGACY


def _current_stream_handle(ordinal: int) -> int:
    """Raw handle of torch's current stream on `ordinal` (the fast path of
    torch.cuda.current_stream(o).cuda_stream; per-run host overhead matters
    for small programs)."""
    import torch
    try:
        h = torch._C._cuda_getCurrentRawStream(ordinal)
    except AttributeError:  # pragma: no cover - older torch
        h = torch.cuda.current_stream(ordinal).cuda_stream
    return h if h else _CUDA_STREAM_LEGACY


class Context:
    """Owns the per-GPU heaps (slot buffers + barrier flags) of K slots."""

    def __init__(self, handle: ctypes.c_void_p, K: int, slot_ordinal: dict, max_bytes: int,
                 group=None):
        self._h = handle
        self.K = K
        self.max_bytes = max_bytes
        self.slot_ordinal = slot_ordinal  # hosted slot -> CUDA ordinal
        self.group = group
        n = ctypes.c_int(0)
        ords = (ctypes.c_int * nat.RS_MAX_RANKS)()
        nat.check(nat.lib().rs_ctx_local_ranks(self._h, ctypes.byref(n), ords))
        self.local_ordinals = [ords[i] for i in range(n.value)]

    # construction
    @classmethod
    def local(cls, K: int, cuda_ordinals: Optional[Sequence[int]] = None, max_bytes: int = 1 << 20):
        if cuda_ordinals is None:
            cuda_ordinals = [0] * K
        h = ctypes.c_void_p()
        nat.check(nat.lib().rs_ctx_create(K, nat.int_array(cuda_ordinals), int(max_bytes), ctypes.byref(h)))
        return cls(h, K, {d: cuda_ordinals[d] for d in range(K)}, max_bytes)

    @classmethod
    def emulated(cls, K: int, slot_rank: Sequence[int], world: int, device: int = 0, max_bytes: int = 1 << 20):
        """Validation mode: `world` ranks emulated on one GPU (own heaps, every
        phase one cooperative launch over all ranks) — the cross-rank kernels
        without several GPUs (rs_ctx_create_emulated)."""
        h = ctypes.c_void_p()
        nat.check(nat.lib().rs_ctx_create_emulated(K, nat.int_array(slot_rank), world, device, int(max_bytes),
                                                   ctypes.byref(h)))
        return cls(h, K, {d: device for d in range(K)}, max_bytes)

    @classmethod
    def virtual(cls, K: int, slot_rank: Sequence[int], world: int):
        """Planning-only context (no GPU): plans can be described, not run."""
        h = ctypes.c_void_p()
        nat.check(nat.lib().rs_ctx_create_virtual(K, nat.int_array(slot_rank), world, ctypes.byref(h)))
        return cls(h, K, {}, 0)

    @classmethod
    def from_process_group(cls, K: int, slot_rank: Sequence[int], max_bytes: int, *, group=None,
                           device: Optional[int] = None):
        import torch
        import torch.distributed as dist
        rank, world = dist.get_rank(group), dist.get_world_size(group)
        if device is None:
            device = torch.cuda.current_device()
        h = ctypes.c_void_p()
        nat.check(nat.lib().rs_ctx_create_rank(K, nat.int_array(slot_rank), world, rank, device,
                                               int(max_bytes), ctypes.byref(h)))
        blob = (ctypes.c_ubyte * nat.RS_IPC_HANDLE_BYTES)()
        nat.check(nat.lib().rs_ctx_ipc_handle(h, blob))
        gathered = [None] * world
        dist.all_gather_object(gathered, bytes(blob), group=group)
        allh = b"".join(gathered)
        nat.check(nat.lib().rs_ctx_open_peers(h, ctypes.c_char_p(allh)))
        dist.barrier(group=group)
        ctx = cls(h, K, {d: device for d in range(K) if slot_rank[d] == rank}, max_bytes, group=group)

        # Host all-gather for collective multicast (NVLS) setup during compiles.
        def _exchange(send, nbytes, recv, _user):
            try:
                out = [None] * world
                dist.all_gather_object(out, ctypes.string_at(send, nbytes), group=group)
                blob = b"".join(out)
                ctypes.memmove(recv, blob, len(blob))
                return 0
            except Exception:  # pragma: no cover - reported as a status by the library
                return 1

        ctx._exchange_cb = nat.EXCHANGE_FN(_exchange)
        nat.check(nat.lib().rs_ctx_set_exchange(h, ctx._exchange_cb, None))
        return ctx

    @property
    def nvls(self) -> bool:
        v = ctypes.c_int(0)
        nat.check(nat.lib().rs_ctx_nvls(self._h, ctypes.byref(v)))
        return bool(v.value)

    def close(self):
        if self._h:
            nat.check(nat.lib().rs_ctx_destroy(self._h))
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # buffers
    def buffer_ptr(self, slot: int) -> int:
        p = ctypes.c_void_p()
        nat.check(nat.lib().rs_ctx_buffer(self._h, slot, ctypes.byref(p)))
        return p.value

    def buffer(self, slot: int, numel: int, dtype="f32"):
        """torch tensor aliasing slot `slot`'s executor buffer (zero copy)."""
        name = {nat.RS_F32: "f32", nat.RS_BF16: "bf16", nat.RS_I32: "i32"}[dtype_code(dtype)]
        if numel * ELEM_BYTES[dtype_code(dtype)] > self.max_bytes:
            raise ValueError("view larger than max_bytes")
        return device_tensor(self.buffer_ptr(slot), numel, name, self.slot_ordinal[slot])

    def buffer_bytes(self, slot: int, nbytes: int):
        """uint8 torch tensor aliasing the first `nbytes` of slot `slot`."""
        if nbytes > self.max_bytes:
            raise ValueError("view larger than max_bytes")
        return device_tensor(self.buffer_ptr(slot), nbytes, "u8", self.slot_ordinal[slot])

    def write(self, slot: int, array: np.ndarray):
        """Copies a host numpy array into the start of slot `slot`'s buffer."""
        import torch
        raw = np.ascontiguousarray(array).view(np.uint8).reshape(-1)
        self.buffer_bytes(slot, raw.size).copy_(torch.from_numpy(raw))

    def read(self, slot: int, nbytes: int) -> np.ndarray:
        return self.buffer_bytes(slot, nbytes).cpu().numpy()

    def _host(self, buf):
        if isinstance(buf, np.ndarray):
            return buf.ctypes.data, buf.nbytes
        return buf.data_ptr(), buf.numel() * buf.element_size()

    def _stream_of(self, slot, stream):
        if stream is not None:
            return stream
        import torch
        return _stream_handle(torch.cuda.current_stream(self.slot_ordinal[slot]))

    def upload(self, slot: int, host, stream=None):
        """Async H2D copy (C-ABI rs_ctx_upload) of a host buffer (pinned
        torch tensor or numpy array) into slot `slot`."""
        ptr, n = self._host(host)
        nat.check(nat.lib().rs_ctx_upload(self._h, slot, ctypes.c_void_p(ptr), n,
                                          ctypes.c_void_p(self._stream_of(slot, stream))))

    def download(self, slot: int, host, stream=None):
        """Async D2H copy (C-ABI rs_ctx_download) of slot `slot` into `host`."""
        ptr, n = self._host(host)
        nat.check(nat.lib().rs_ctx_download(self._h, slot, ctypes.c_void_p(ptr), n,
                                            ctypes.c_void_p(self._stream_of(slot, stream))))

    @property
    def hosted_slots(self):
        return sorted(self.slot_ordinal)

    def set_option(self, key: str, value: int):
        """Context knobs for later compiles: push_min_bytes (-1 = never push),
        barrier_timeout_ms, nvls, nvls_min_group, nvls_min_bytes, ll_max_bytes
        (one-shot budget per GPU pair and step; 0 = never)."""
        nat.check(nat.lib().rs_ctx_set_option(self._h, key.encode(), int(value)))

    def synchronize(self):
        import torch
        for o in self.local_ordinals:
            torch.cuda.synchronize(o)
        nat.check(nat.lib().rs_ctx_synchronize(self._h))

    def compile(self, program: LoweredProgram, elems: int, dtype="f32") -> "Plan":
        return Plan(self, program, elems, dtype)


class Plan:
    """A compiled program: per-step, per-GPU task lists resident on device."""

    def __init__(self, ctx: Context, program: LoweredProgram, elems: int, dtype="f32"):
        self.ctx = ctx
        self.program = program
        self.elems = int(elems)
        self.dtype = dtype_code(dtype)
        ops, sgp, gmp, mem = program.to_csr()
        p32 = ctypes.POINTER(ctypes.c_int32)
        h = ctypes.c_void_p()
        nat.check(nat.lib().rs_plan_compile(ctx._h, len(program.steps), ops.ctypes.data_as(p32),
                                            sgp.ctypes.data_as(p32), gmp.ctypes.data_as(p32),
                                            mem.ctypes.data_as(p32), self.elems, self.dtype,
                                            ctypes.byref(h)))
        self._h = h
        self._run_fn = nat.lib().rs_plan_run
        self._stream_key = None
        self._stream_arr = None

    def close(self):
        if self._h:
            nat.lib().rs_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _streams(self, streams):
        if streams is None:
            key = tuple(_current_stream_handle(o) for o in self.ctx.local_ordinals)
        else:
            key = tuple(streams)
        if key != self._stream_key:  # cached: the common case is the same stream every run
            self._stream_arr = (ctypes.c_void_p * max(1, len(key)))(*[ctypes.c_void_p(s) for s in key])
            self._stream_key = key
        return self._stream_arr

    def run(self, bufs=None, streams=None):
        """Enqueue. bufs=None: in place on the context buffers; else K device
        pointers or tensors (slot-indexed) copied in and out."""
        arr = None
        if bufs is not None:
            ptrs = [b if isinstance(b, int) else (b.data_ptr() if b is not None else 0) for b in bufs]
            arr = (ctypes.c_void_p * self.ctx.K)(*[ctypes.c_void_p(p) for p in ptrs])
        code = self._run_fn(self._h, arr, self._streams(streams))
        if code:
            nat.check(code)

    def run_host(self, host_bufs, streams=None):
        """End to end from host memory: H2D copy-in, program, D2H copy-out."""
        ptrs = []
        for b in host_bufs:
            if b is None:
                ptrs.append(0)
            elif isinstance(b, np.ndarray):
                ptrs.append(b.ctypes.data)
            else:
                ptrs.append(b.data_ptr())
        arr = (ctypes.c_void_p * self.ctx.K)(*[ctypes.c_void_p(p) for p in ptrs])
        nat.check(nat.lib().rs_plan_run_host(self._h, arr, self._streams(streams)))

    @property
    def launches(self) -> int:
        n = ctypes.c_int(0)
        nat.check(nat.lib().rs_plan_launch_count(self._h, ctypes.byref(n)))
        return n.value

    def step_bytes(self, step: int):
        """(max per-rank link bytes per direction, max per-rank HBM bytes)."""
        a, b = ctypes.c_double(), ctypes.c_double()
        nat.check(nat.lib().rs_plan_step_bytes(self._h, step, ctypes.byref(a), ctypes.byref(b)))
        return a.value, b.value

    def time_us(self, warmup: int = 1, iters: int = 5) -> float:
        """Device time of one run (rs_plan_time: back-to-back runs bracketed by
        CUDA events on every local GPU's stream, slowest GPU). Synchronous."""
        us = ctypes.c_double()
        nat.check(nat.lib().rs_plan_time(self._h, int(warmup), int(iters), ctypes.byref(us)))
        return us.value

    def predict_us(self, launch_us: float = 8.0, link_gbs: float = 650.0, hbm_gbs: float = 6000.0) -> float:
        """B200-calibrated cost of one run from the plan's own traffic
        (rs_plan_predict_us); defaults = measured per-step latency (K=4),
        P2P AllReduce link rate and local step kernel HBM rate."""
        us = ctypes.c_double()
        nat.check(nat.lib().rs_plan_predict_us(self._h, float(launch_us), float(link_gbs), float(hbm_gbs),
                                               ctypes.byref(us)))
        return us.value

    def describe(self) -> dict:
        """The compiled plan: per step, per rank, entry-barrier ranks and tasks."""
        import json
        out = ctypes.c_void_p()
        nat.check(nat.lib().rs_plan_describe_json(self._h, ctypes.byref(out)))
        return json.loads(nat.take_string(out))

    def set_launch(self, max_ctas: int = 0, threads: int = 0):
        nat.check(nat.lib().rs_plan_set_launch(self._h, int(max_ctas), int(threads)))

    def set_option(self, key: str, value: int):
        """Named plan knobs (include/redsynth_exec.h rs_plan_set_option):
        unroll (4|8), threads, max_ctas, wide_loads, dynamic_pieces, pdl,
        local_wide, vec256, remote256, piece_queue (0|1|2)."""
        nat.check(nat.lib().rs_plan_set_option(self._h, key.encode(), int(value)))
