// The sm_100a step kernel: one launch per (program step, rank).
//
// A step of a lowered program is compiled (plan.cc) into "tasks": byte
// ranges that one owner produces by summing its sources in group order and
// storing the result to every destination. Sources and destinations are
// slot buffers on this GPU or on NVSwitch peers (mapped peer pointers), so a
// single pass covers every collective of /root/reference/proj/src/
// semantics.cc:259-310:
//   AllReduce      owner m: its 1/n slice of R, sources = all members,
//                  destinations = all members (reduce-scatter + all-gather
//                  fused into one pull-sum-push pass, 2(n-1)/n per link)
//   ReduceScatter  owner m: run m of R, pull-sum into its own buffer
//   Reduce         owners = non-roots, slices of R, sum -> root only
//   AllGather /    owners = the receivers, each pulls a slice of a row from
//   Broadcast      its holder and fans it out to the other receivers
// Small steps run one-shot (LL): every destination sums its own result from
// flagged 16-byte packets its sources pushed into its LL area (kModeLL).
// Large AllReduce groups on >= 4 GPUs may use NVLS multimem instead.
// Memory: 16-byte vector loads (ld.global.nc.L1::no_allocate on one GPU,
// weak ld.global.L1::no_allocate across GPUs) and streaming
// stores, 4 (cross-GPU) or 8 (one GPU) vectors in flight per thread per
// source, coalesced 512 B per warp.
// Inter-GPU ordering: epoch flags in each rank's heap (relaxed st.sys behind
// one fence.acq_rel.sys per CTA; ld.acquire.sys spins); no NCCL, no host
// synchronisation between steps.
#include <cuda_bf16.h>
#include <cuda_runtime.h>

#include <cstdio>

#include "device_types.h"

namespace rs {
namespace {

// Streaming 16-byte load. The non-coherent (.nc) form is only legal for data
// that is read-only for the kernel's whole lifetime: true in a single-rank
// context (every step of a local plan is hazard-free and nobody else writes
// the heap), not across GPUs, where a peer may write a slot buffer (previous
// step's results) while this kernel waits at its entry barrier. Cross-rank
// launches therefore use weak ld.global (ordered after the entry acquire by
// the CTA barrier), still without L1 allocation.
template <bool kNc>
__device__ __forceinline__ uint4 LoadStream(const void* p) {
  uint4 v;
#ifndef RS_LOAD_QUAL
// 256-byte L2 prefetch on the streaming loads: neutral to +2 % on one GPU
// depending on the box, neutral over NVLink (profiles/r01_l2_prefetch_ab.txt).
#define RS_LOAD_QUAL ".L1::no_allocate.L2::256B"
#endif
  if constexpr (kNc) {
    asm volatile("ld.global.nc" RS_LOAD_QUAL ".v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p));
  } else {
    asm volatile("ld.global" RS_LOAD_QUAL ".v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(p)
                 : "memory");
  }
  return v;
}

// L2-coherent load (skips L1): data a peer GPU pushed during this kernel,
// read after an acquire of its chunk flag.
__device__ __forceinline__ uint4 LoadCoherent(const void* p) {
  uint4 v;
  asm volatile("ld.global.cg.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void Store(void* p, const uint4& v) {
#ifndef RS_STORE_QUAL
// Streaming stores: measured +2% HBM efficiency in local mode over plain
// st.global (profiles/r01_store_hint_ab.txt); .cs measured the same.
#define RS_STORE_QUAL ".L1::no_allocate"
#endif
  asm volatile("st.global" RS_STORE_QUAL ".v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}

__device__ __forceinline__ uint64_t LoadAcquireSys(const uint64_t* p) {
  uint64_t v;
  asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void StoreReleaseSys(uint64_t* p, uint64_t v) {
  asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void StoreRelaxedSys(uint64_t* p, uint64_t v) {
  asm volatile("st.relaxed.sys.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ void FenceSys() { asm volatile("fence.acq_rel.sys;" ::: "memory"); }

// Flag stores: RS_SYNC_STRICT=1 restores release stores behind extra fences
// (A/B of the barrier cost); the default orders data before flags with one
// system fence per CTA plus one in the last CTA, then relaxed flag stores.
#ifndef RS_SYNC_STRICT
#define RS_SYNC_STRICT 0
#endif
__device__ __forceinline__ void SignalStore(uint64_t* p, uint64_t v) {
  if (RS_SYNC_STRICT) StoreReleaseSys(p, v);
  else StoreRelaxedSys(p, v);
}

__device__ __forceinline__ uint64_t GlobalTimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ bool Failed(const int* error_flag) {
  return *reinterpret_cast<const volatile int*>(error_flag) != 0;
}

// Checked builds (make checked, RS_CHECKED): device-side bounds and protocol
// assertions. A failed check prints once per CTA and raises the rank's error
// flag with a code >= 2 (never a trap), which rs_ctx_synchronize reports.
enum : int { kCheckRange = 2, kCheckLLFuture = 3, kCheckFlagFuture = 4, kCheckPiece = 5 };
#ifdef RS_CHECKED
__device__ __noinline__ void CheckFail(int* error_flag, int code, uint64_t x, uint64_t y) {
  if (atomicCAS(error_flag, 0, code) == 0)
    printf("redsynth checked build: assertion %d failed (block %d thread %d): %llu vs %llu\n", code, blockIdx.x,
           threadIdx.x, static_cast<unsigned long long>(x), static_cast<unsigned long long>(y));
}
#define RS_CHECK(cond, flag, code, x, y)                  \
  do {                                                    \
    if (!(cond)) CheckFail((flag), (code), (x), (y));     \
  } while (0)
#else
#define RS_CHECK(cond, flag, code, x, y) \
  do {                                   \
  } while (0)
#endif

// Spin until *flag >= target; on timeout raise the error flag and give up
// (the data is then wrong, but the GPU is not hung; the host reports it).
// Once this rank's error flag is up every later wait returns at once, so a
// dead peer costs one timeout per run, not one per wait.
__device__ void WaitAtLeast(const uint64_t* flag, uint64_t target, uint64_t timeout_ns,
                            int* error_flag) {
  // Tight spin first (a peer is usually < 2 us away), then back off.
  for (int i = 0; i < 4096; ++i) {
    if (LoadAcquireSys(flag) >= target) return;
  }
  if (Failed(error_flag)) return;
  const uint64_t t0 = GlobalTimer();
  while (LoadAcquireSys(flag) < target) {
    if (Failed(error_flag)) return;
    if (GlobalTimer() - t0 > timeout_ns) {
      atomicExch(error_flag, 1);
      return;
    }
    __nanosleep(64);
  }
}

// ---- element arithmetic -----------------------------------------------

// f32: IEEE adds in source order (no FMA possible: adds only).
struct F32Acc {
  float v[4];
  __device__ __forceinline__ void Init(const uint4& r) {
    v[0] = __uint_as_float(r.x); v[1] = __uint_as_float(r.y);
    v[2] = __uint_as_float(r.z); v[3] = __uint_as_float(r.w);
  }
  __device__ __forceinline__ void Add(const uint4& r) {
    v[0] = __fadd_rn(v[0], __uint_as_float(r.x)); v[1] = __fadd_rn(v[1], __uint_as_float(r.y));
    v[2] = __fadd_rn(v[2], __uint_as_float(r.z)); v[3] = __fadd_rn(v[3], __uint_as_float(r.w));
  }
  __device__ __forceinline__ uint4 Pack() const {
    return make_uint4(__float_as_uint(v[0]), __float_as_uint(v[1]), __float_as_uint(v[2]),
                      __float_as_uint(v[3]));
  }
};

// bf16: widen to f32, add in source order, round to nearest even once.
struct BF16Acc {
  float v[8];
  __device__ __forceinline__ static void Widen(uint32_t w, float& lo, float& hi) {
    lo = __uint_as_float(w << 16);
    hi = __uint_as_float(w & 0xffff0000u);
  }
  __device__ __forceinline__ void Init(const uint4& r) {
    Widen(r.x, v[0], v[1]); Widen(r.y, v[2], v[3]); Widen(r.z, v[4], v[5]); Widen(r.w, v[6], v[7]);
  }
  __device__ __forceinline__ void Add(const uint4& r) {
    float t[8];
    Widen(r.x, t[0], t[1]); Widen(r.y, t[2], t[3]); Widen(r.z, t[4], t[5]); Widen(r.w, t[6], t[7]);
#pragma unroll
    for (int i = 0; i < 8; ++i) v[i] = __fadd_rn(v[i], t[i]);
  }
  __device__ __forceinline__ static uint32_t Narrow(float lo, float hi) {
    __nv_bfloat162 p = __floats2bfloat162_rn(lo, hi);  // cvt.rn.bf16x2.f32
    return *reinterpret_cast<uint32_t*>(&p);
  }
  __device__ __forceinline__ uint4 Pack() const {
    return make_uint4(Narrow(v[0], v[1]), Narrow(v[2], v[3]), Narrow(v[4], v[5]),
                      Narrow(v[6], v[7]));
  }
};

// i32: two's-complement wrapping adds.
struct I32Acc {
  uint32_t v[4];
  __device__ __forceinline__ void Init(const uint4& r) { v[0] = r.x; v[1] = r.y; v[2] = r.z; v[3] = r.w; }
  __device__ __forceinline__ void Add(const uint4& r) { v[0] += r.x; v[1] += r.y; v[2] += r.z; v[3] += r.w; }
  __device__ __forceinline__ uint4 Pack() const { return make_uint4(v[0], v[1], v[2], v[3]); }
};

template <int DT> struct AccOf;
template <> struct AccOf<RS_F32> { using T = F32Acc; };
template <> struct AccOf<RS_BF16> { using T = BF16Acc; };
template <> struct AccOf<RS_I32> { using T = I32Acc; };

// One block-wide chunk: bytes [begin, end) of the task, 16-byte aligned;
// thread t handles vectors begin + (u * blockDim + t) * 16, u < kUnroll.
template <int DT, int kUnroll, bool kNc, bool kCoherent = false>
__device__ __forceinline__ void VectorChunk(const Task& t, void* const* ptrs, uint64_t begin,
                                            uint64_t end) {
  using Acc = typename AccOf<DT>::T;
  uint64_t off[kUnroll];
  bool ok[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    off[u] = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    ok[u] = off[u] < end;
  }
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  uint4 raw[kUnroll] = {};
  const char* s0 = static_cast<const char*>(src[0]);
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    if (ok[u]) raw[u] = kCoherent ? LoadCoherent(s0 + off[u]) : LoadStream<kNc>(s0 + off[u]);
  if (t.nsrc > 1) {
    Acc acc[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) acc[u].Init(raw[u]);
    for (int i = 1; i < t.nsrc; ++i) {
      const char* si = static_cast<const char*>(src[i]);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (ok[u]) raw[u] = kCoherent ? LoadCoherent(si + off[u]) : LoadStream<kNc>(si + off[u]);
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) acc[u].Add(raw[u]);
    }
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) raw[u] = acc[u].Pack();
  }
  for (int j = 0; j < t.ndst; ++j) {
    char* d = static_cast<char*>(dst[j]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (ok[u]) Store(d + off[u], raw[u]);
  }
}

// 256-bit streaming load / store (sm_100): 32 bytes per thread per
// instruction. Single-rank (local) launches only: non-coherent loads.
struct Vec32 {
  uint4 lo, hi;
};

__device__ __forceinline__ Vec32 LoadStream32(const void* p) {
  Vec32 v;
  asm volatile("ld.global.nc" RS_LOAD_QUAL ".v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                 "=r"(v.hi.w)
               : "l"(p));
  return v;
}

__device__ __forceinline__ void Store32(void* p, const Vec32& v) {
  asm volatile("st.global" RS_STORE_QUAL ".v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(p), "r"(v.lo.x),
               "r"(v.lo.y), "r"(v.lo.z), "r"(v.lo.w), "r"(v.hi.x), "r"(v.hi.y), "r"(v.hi.z), "r"(v.hi.w)
               : "memory");
}

// One-GPU copy chunk (a single source: the AllGather / Broadcast tasks, the
// write-heavy steps) with 256-bit vectors: thread t handles 32-byte vectors
// begin + (u * blockDim + t) * 32, u < kU. Measured on a 1-read / 3-write
// copy at 148 x 512 threads: 6.16 TB/s vs 4.83 with 128-bit vectors
// (tools/hbm_write_probe.cu, profiles/r02_hbm_write_probe.txt). Sums keep
// the 128-bit path (their f32 accumulators would not fit beside 256-bit
// batches; they are read-heavy and already near the HBM rate).
template <int kU>
__device__ __forceinline__ void CopyChunk32(const Task& t, void* const* ptrs, uint64_t begin, uint64_t end) {
  // task fields as locals: the stores' "memory" clobber would reload them per loop
  const int nsrc = t.nsrc, ndst = t.ndst;
  uint64_t off[kU];
  bool ok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    off[u] = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 32u;
    ok[u] = off[u] < end;
  }
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + nsrc;
  Vec32 raw[kU];
  const char* s0 = static_cast<const char*>(src[0]);
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    raw[u] = Vec32{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};  // defined on every path (no spills)
    if (ok[u]) raw[u] = LoadStream32(s0 + off[u]);
  }
  for (int j = 0; j < ndst; ++j) {
    char* d = static_cast<char*>(dst[j]);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (ok[u]) Store32(d + off[u], raw[u]);
  }
}

// Weak (coherent-after-acquire) 256-bit load for cross-GPU sources.
__device__ __forceinline__ Vec32 LoadWeak32(const void* p) {
  Vec32 v;
  asm volatile("ld.global" RS_LOAD_QUAL ".v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                 "=r"(v.hi.w)
               : "l"(p)
               : "memory");
  return v;
}

__device__ __forceinline__ Vec32 LoadCoherent32(const void* p) {
  Vec32 v;
  asm volatile("ld.global.cg.v8.b32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=r"(v.lo.x), "=r"(v.lo.y), "=r"(v.lo.z), "=r"(v.lo.w), "=r"(v.hi.x), "=r"(v.hi.y), "=r"(v.hi.z),
                 "=r"(v.hi.w)
               : "l"(p));
  return v;
}

// Cross-GPU copy with 256-bit vectors (push landing pieces): kU 32-byte
// vectors per thread, weak loads.
template <int kU>
__device__ __forceinline__ void RemoteCopyChunk32(const Task& t, void* const* ptrs, uint64_t begin, uint64_t end) {
  uint64_t off[kU];
  bool ok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    off[u] = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 32u;
    ok[u] = off[u] < end;
  }
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  Vec32 raw[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    raw[u] = Vec32{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    if (ok[u]) raw[u] = LoadWeak32(static_cast<const char*>(src[0]) + off[u]);
  }
  for (int j = 0; j < t.ndst; ++j) {
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (ok[u]) Store32(static_cast<char*>(dst[j]) + off[u], raw[u]);
  }
}

// Cross-GPU sum with 256-bit vectors and every source in flight (option
// remote256, default on): one 32-byte vector per thread per source; kCoherent
// for push reductions over landed scratch (written during this kernel).
template <int DT, int kS, bool kCoherent = false>
__device__ __forceinline__ void WideChunk32(const Task& t, void* const* ptrs, uint64_t begin, uint64_t end) {
  using Acc = typename AccOf<DT>::T;
  const uint64_t off = begin + static_cast<uint64_t>(threadIdx.x) * 32u;
  if (off >= end) return;
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  Vec32 raw[kS];
#pragma unroll
  for (int i = 0; i < kS; ++i) {
    raw[i] = Vec32{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    if (i < t.nsrc)
      raw[i] = kCoherent ? LoadCoherent32(static_cast<const char*>(src[i]) + off)
                         : LoadWeak32(static_cast<const char*>(src[i]) + off);
  }
  Acc lo, hi;
  lo.Init(raw[0].lo);
  hi.Init(raw[0].hi);
#pragma unroll
  for (int i = 1; i < kS; ++i) {
    if (i < t.nsrc) {
      lo.Add(raw[i].lo);
      hi.Add(raw[i].hi);
    }
  }
  const Vec32 out{lo.Pack(), hi.Pack()};
  for (int j = 0; j < t.ndst; ++j) Store32(static_cast<char*>(dst[j]) + off, out);
}

// One-GPU sum chunk with 256-bit vectors (A/B: vec256 = 2): as
// VectorChunk<DT, 2 kU> but 32 bytes per memory instruction.
template <int DT, int kU>
__device__ __forceinline__ void SumChunk32(const Task& t, void* const* ptrs, uint64_t begin, uint64_t end) {
  // task fields as locals: the stores' "memory" clobber would reload them per loop
  const int nsrc = t.nsrc, ndst = t.ndst;
  using Acc = typename AccOf<DT>::T;
  uint64_t off[kU];
  bool ok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    off[u] = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 32u;
    ok[u] = off[u] < end;
  }
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + nsrc;
  Vec32 raw[kU];
  const char* s0 = static_cast<const char*>(src[0]);
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    raw[u] = Vec32{make_uint4(0, 0, 0, 0), make_uint4(0, 0, 0, 0)};
    if (ok[u]) raw[u] = LoadStream32(s0 + off[u]);
  }
  Acc acc[2 * kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    acc[2 * u].Init(raw[u].lo);
    acc[2 * u + 1].Init(raw[u].hi);
  }
  for (int i = 1; i < nsrc; ++i) {
    const char* si = static_cast<const char*>(src[i]);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (ok[u]) raw[u] = LoadStream32(si + off[u]);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      acc[2 * u].Add(raw[u].lo);
      acc[2 * u + 1].Add(raw[u].hi);
    }
  }
#pragma unroll
  for (int u = 0; u < kU; ++u) raw[u] = Vec32{acc[2 * u].Pack(), acc[2 * u + 1].Pack()};
  for (int j = 0; j < ndst; ++j) {
    char* d = static_cast<char*>(dst[j]);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (ok[u]) Store32(d + off[u], raw[u]);
  }
}

// Cross-GPU pull chunk with every source's loads in flight at once: all
// nsrc (<= kS) sources' kU vectors are loaded before the first add, so a
// chunk costs one round trip instead of nsrc serialized ones; the sum is
// still taken in source (group) order. Remote loads are weak ld.global.
template <int DT, int kS, int kU, bool kCoherent = false, bool kNc = false>
__device__ __forceinline__ void VectorChunkWide(const Task& t, void* const* ptrs, uint64_t begin,
                                                uint64_t end) {
  using Acc = typename AccOf<DT>::T;
  uint64_t off[kU];
  bool ok[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) {
    off[u] = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    ok[u] = off[u] < end;
  }
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  uint4 raw[kS][kU];
#pragma unroll
  for (int i = 0; i < kS; ++i) {
#pragma unroll
    for (int u = 0; u < kU; ++u) raw[i][u] = make_uint4(0, 0, 0, 0);
    if (i < t.nsrc) {
      const char* si = static_cast<const char*>(src[i]);
#pragma unroll
      for (int u = 0; u < kU; ++u)
        if (ok[u]) raw[i][u] = kCoherent ? LoadCoherent(si + off[u]) : LoadStream<kNc>(si + off[u]);
    }
  }
  Acc acc[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) acc[u].Init(raw[0][u]);
#pragma unroll
  for (int i = 1; i < kS; ++i) {
    if (i < t.nsrc) {
#pragma unroll
      for (int u = 0; u < kU; ++u) acc[u].Add(raw[i][u]);
    }
  }
  uint4 out[kU];
#pragma unroll
  for (int u = 0; u < kU; ++u) out[u] = acc[u].Pack();
  for (int j = 0; j < t.ndst; ++j) {
    char* d = static_cast<char*>(dst[j]);
#pragma unroll
    for (int u = 0; u < kU; ++u)
      if (ok[u]) Store(d + off[u], out[u]);
  }
}

// NVLS AllReduce chunk: the NVSwitch sums the group's copies
// (multimem.ld_reduce on the multicast address; bf16 accumulates in f32) and
// multimem.st writes the result to every member. f32 / bf16 only.
template <int DT, int kUnroll>
__device__ __forceinline__ void NvlsChunk(const Task& t, void* const* ptrs, uint64_t begin,
                                          uint64_t end) {
  char* mc = static_cast<char*>(ptrs[t.ptr_begin]);
  uint4 v[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    v[u] = make_uint4(0, 0, 0, 0);  // defined on every path (no spills around the loads)
    const uint64_t off = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    if (off >= end) continue;
    if constexpr (DT == RS_BF16) {
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(mc + off)
                   : "memory");
    } else {
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(mc + off)
                   : "memory");
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t off = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    if (off >= end) continue;
    if constexpr (DT == RS_BF16) {
      asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(mc + off),
                   "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                   : "memory");
    } else {
      asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + off),
                   "r"(v[u].x), "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                   : "memory");
    }
  }
}

// NVLS Reduce chunk: the switch sums the group's copies of the range and the
// owner stores the result to its destinations (the root) with ordinary
// stores. f32 / bf16 only.
template <int DT, int kUnroll>
__device__ __forceinline__ void NvlsReduceChunk(const Task& t, void* const* ptrs, uint64_t begin,
                                                uint64_t end) {
  const char* mc = static_cast<const char*>(ptrs[t.ptr_begin]);
  void* const* dst = ptrs + t.ptr_begin + 1;
  uint4 v[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    v[u] = make_uint4(0, 0, 0, 0);
    const uint64_t off = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    if (off >= end) continue;
    if constexpr (DT == RS_BF16) {
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(mc + off)
                   : "memory");
    } else {
      asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                   : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                   : "l"(mc + off)
                   : "memory");
    }
  }
  for (int j = 0; j < t.ndst; ++j) {
    char* d = static_cast<char*>(dst[j]);
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint64_t off = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
      if (off < end) Store(d + off, v[u]);
    }
  }
}

// NVLS Broadcast chunk: weak loads of the root's data, one store per vector
// to the multicast address (the switch replicates it into every member).
template <int kUnroll>
__device__ __forceinline__ void NvlsBroadcastChunk(const Task& t, void* const* ptrs, uint64_t begin,
                                                   uint64_t end) {
  const char* src = static_cast<const char*>(ptrs[t.ptr_begin]);
  char* mc = static_cast<char*>(ptrs[t.ptr_begin + 1]);
  uint4 v[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    v[u] = make_uint4(0, 0, 0, 0);
    const uint64_t off = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    if (off < end) v[u] = LoadStream<false>(src + off);
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint64_t off = begin + (static_cast<uint64_t>(u) * blockDim.x + threadIdx.x) * 16u;
    if (off >= end) continue;
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + off), "r"(v[u].x),
                 "r"(v[u].y), "r"(v[u].z), "r"(v[u].w)
                 : "memory");
  }
}

__device__ __forceinline__ void FenceProxyAlias() { asm volatile("fence.proxy.alias;" ::: "memory"); }

// A scalar task (< 16 bytes): one element per thread.
template <int DT>
__device__ void ScalarTask(const Task& t, void* const* ptrs) {
  constexpr int kEs = DT == RS_BF16 ? 2 : 4;
  const uint64_t x = t.lo + static_cast<uint64_t>(threadIdx.x) * kEs;
  if (x >= t.hi) return;
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  if (DT == RS_BF16) {
    const uint16_t first = *reinterpret_cast<const uint16_t*>(static_cast<const char*>(src[0]) + x);
    uint16_t out = first;
    if (t.nsrc > 1) {
      float acc = __uint_as_float(static_cast<uint32_t>(first) << 16);
      for (int i = 1; i < t.nsrc; ++i) {
        const uint16_t h = *reinterpret_cast<const uint16_t*>(static_cast<const char*>(src[i]) + x);
        acc = __fadd_rn(acc, __uint_as_float(static_cast<uint32_t>(h) << 16));
      }
      __nv_bfloat16 b = __float2bfloat16_rn(acc);
      out = *reinterpret_cast<uint16_t*>(&b);
    }
    for (int j = 0; j < t.ndst; ++j) *reinterpret_cast<uint16_t*>(static_cast<char*>(dst[j]) + x) = out;
  } else {
    uint32_t out = *reinterpret_cast<const uint32_t*>(static_cast<const char*>(src[0]) + x);
    for (int i = 1; i < t.nsrc; ++i) {
      const uint32_t w = *reinterpret_cast<const uint32_t*>(static_cast<const char*>(src[i]) + x);
      if (DT == RS_F32) out = __float_as_uint(__fadd_rn(__uint_as_float(out), __uint_as_float(w)));
      else out += w;
    }
    for (int j = 0; j < t.ndst; ++j) *reinterpret_cast<uint32_t*>(static_cast<char*>(dst[j]) + x) = out;
  }
}

// ---- one-shot (LL) tasks -------------------------------------------------

__device__ __forceinline__ void StoreLL(char* p, uint2 d, uint32_t flag) {
  asm volatile("st.volatile.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(d.x), "r"(flag), "r"(d.y),
               "r"(flag)
               : "memory");
}

// Waits for the packet at p to carry `flag` in both halves (each 8-byte half
// {data, flag} lands atomically), returns its payload.
__device__ __forceinline__ uint2 LoadLL(const char* p, uint32_t flag, uint64_t timeout_ns, int* error_flag) {
  uint32_t d0, f0, d1, f1;
  uint64_t t0 = 0;
  for (uint32_t spin = 0;; ++spin) {
    asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(d0), "=r"(f0), "=r"(d1), "=r"(f1)
                 : "l"(p)
                 : "memory");
    if (f0 == flag && f1 == flag) break;
    // a packet of a later epoch in this parity region: the sender ran two
    // epochs ahead and overwrote data not yet consumed
    RS_CHECK(static_cast<int32_t>(f0 - flag) <= 0 && static_cast<int32_t>(f1 - flag) <= 0, error_flag,
             kCheckLLFuture, f0, flag);
    if (spin == 4096) {
      if (Failed(error_flag)) break;
      t0 = GlobalTimer();
    }
    if (spin > 4096 && (spin & 63) == 0 && (Failed(error_flag) || GlobalTimer() - t0 > timeout_ns)) {
      atomicExch(error_flag, 1);
      break;
    }
  }
  return make_uint2(d0, d1);
}

template <int DT>
__device__ __forceinline__ uint2 AddPacket(uint2 a, uint2 b) {
  if constexpr (DT == RS_BF16) {
    return a;  // bf16 sums are kept in f32 by the caller
  } else if constexpr (DT == RS_F32) {
    return make_uint2(__float_as_uint(__fadd_rn(__uint_as_float(a.x), __uint_as_float(b.x))),
                      __float_as_uint(__fadd_rn(__uint_as_float(a.y), __uint_as_float(b.y))));
  } else {
    return make_uint2(a.x + b.x, a.y + b.y);
  }
}

// LL task pointers: the (at most one) untagged source is local.
__device__ __forceinline__ const char* LLLocal(const Task& t, void* const* src) {
  const char* local = nullptr;
  for (int i = 0; i < t.nsrc; ++i)
    if (!(reinterpret_cast<uintptr_t>(src[i]) & 1u)) local = static_cast<const char*>(src[i]);
  return local;
}

// Packets per thread in flight in the one-shot sweeps (memory-level
// parallelism: a thread's packets are independent round trips).
constexpr int kLLBatch = 8;

__device__ __forceinline__ uint4 LoadVolatile16(const char* p) {
  uint4 v;
  asm volatile("ld.volatile.global.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "l"(p)
               : "memory");
  return v;
}

// Sweep 1 over packets [begin, end) (8-byte aligned payload offsets) of an
// LL task: push the local source's packets to every tagged destination.
__device__ __forceinline__ void LLSend(const Task& t, void* const* ptrs, uint64_t begin, uint64_t end,
                                       uint32_t flag, uint64_t parity_off) {
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  const char* local = LLLocal(t, src);
  if (!local) return;
  const uint64_t stride = static_cast<uint64_t>(blockDim.x) * 8u;
  for (uint64_t x0 = begin + static_cast<uint64_t>(threadIdx.x) * 8u; x0 < end; x0 += stride * kLLBatch) {
    uint2 mine[kLLBatch];
#pragma unroll
    for (int b = 0; b < kLLBatch; ++b) {
      const uint64_t x = x0 + b * stride;
      if (x < end) mine[b] = *reinterpret_cast<const uint2*>(local + x);
    }
    for (int j = 0; j < t.ndst; ++j) {
      const uintptr_t d = reinterpret_cast<uintptr_t>(dst[j]);
      if (!(d & 1u)) continue;
      char* base = reinterpret_cast<char*>((d & ~uintptr_t{1}) + parity_off);
#pragma unroll
      for (int b = 0; b < kLLBatch; ++b) {
        const uint64_t x = x0 + b * stride;
        if (x < end) StoreLL(base + 2 * x, mine[b], flag);
      }
    }
  }
}

// Up to kLLWide sources: every source's packets of a batch are loaded before
// any flag is checked, so the sources' latencies overlap (a group of n GPUs
// otherwise pays n-1 dependent local round trips per batch).
constexpr int kLLWide = 4;

template <int DT>
__device__ __forceinline__ void StoreLLResult(const Task& t, void* const* dst, uint64_t x, uint2 out) {
  constexpr uint32_t kEs = DT == RS_BF16 ? 2 : 4;
  const bool whole = x >= t.lo && x + 8 <= t.hi;
  for (int j = 0; j < t.ndst; ++j) {
    const uintptr_t d = reinterpret_cast<uintptr_t>(dst[j]);
    if (d & 1u) continue;
    char* base = reinterpret_cast<char*>(d);
    if (whole) {
      *reinterpret_cast<uint2*>(base + x) = out;
      continue;
    }
    // Edge packet: only the elements inside [lo, hi).
    const char* bytes = reinterpret_cast<const char*>(&out);
    for (uint32_t e = 0; e < 8; e += kEs) {
      if (x + e < t.lo || x + e >= t.hi) continue;
      if (kEs == 2) *reinterpret_cast<uint16_t*>(base + x + e) = *reinterpret_cast<const uint16_t*>(bytes + e);
      else *reinterpret_cast<uint32_t*>(base + x + e) = *reinterpret_cast<const uint32_t*>(bytes + e);
    }
  }
}

template <int DT>
__device__ __forceinline__ void LLReceiveWide(const Task& t, void* const* src, void* const* dst, const char* local,
                                              uint64_t begin, uint64_t end, uint32_t flag, uint64_t parity_off,
                                              uint64_t timeout_ns, int* error_flag) {
  constexpr int kB = 4;  // packets per thread per pass
  const uint64_t stride = static_cast<uint64_t>(blockDim.x) * 8u;
  const int n = t.nsrc;
  const char* base[kLLWide];
#pragma unroll
  for (int i = 0; i < kLLWide; ++i) {
    const uintptr_t s = i < n ? reinterpret_cast<uintptr_t>(src[i]) : 0;
    base[i] = (s & 1u) ? reinterpret_cast<const char*>((s & ~uintptr_t{1}) + parity_off) : nullptr;
  }
  for (uint64_t x0 = begin + static_cast<uint64_t>(threadIdx.x) * 8u; x0 < end; x0 += stride * kB) {
    uint4 pk[kLLWide][kB];
    uint2 mine[kB];
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const uint64_t x = x0 + b * stride;
      mine[b] = (local && x < end) ? *reinterpret_cast<const uint2*>(local + x) : make_uint2(0, 0);
    }
#pragma unroll
    for (int i = 0; i < kLLWide; ++i) {  // every source's loads in flight at once
#pragma unroll
      for (int b = 0; b < kB; ++b) {
        const uint64_t x = x0 + b * stride;
        pk[i][b] = (base[i] && x < end) ? LoadVolatile16(base[i] + 2 * x) : make_uint4(0, flag, 0, flag);
      }
    }
#pragma unroll
    for (int b = 0; b < kB; ++b) {
      const uint64_t x = x0 + b * stride;
      if (x >= end) continue;
      uint2 out = mine[b];
      float f[4];
#pragma unroll
      for (int i = 0; i < kLLWide; ++i) {
        if (i >= n) break;
        uint2 v = mine[b];
        if (base[i]) {
          if (pk[i][b].y != flag || pk[i][b].w != flag) {
            const uint2 late = LoadLL(base[i] + 2 * x, flag, timeout_ns, error_flag);
            pk[i][b] = make_uint4(late.x, flag, late.y, flag);
          }
          v = make_uint2(pk[i][b].x, pk[i][b].z);
        }
        if constexpr (DT == RS_BF16) {
          float g[4];
          BF16Acc::Widen(v.x, g[0], g[1]);
          BF16Acc::Widen(v.y, g[2], g[3]);
#pragma unroll
          for (int k = 0; k < 4; ++k) f[k] = i == 0 ? g[k] : __fadd_rn(f[k], g[k]);
        }
        out = i == 0 ? v : AddPacket<DT>(out, v);
      }
      if constexpr (DT == RS_BF16) {
        if (n > 1) out = make_uint2(BF16Acc::Narrow(f[0], f[1]), BF16Acc::Narrow(f[2], f[3]));
      }
      StoreLLResult<DT>(t, dst, x, out);
    }
  }
}

// Sweep 2 over the same packets (same thread per packet, so a task that sends
// its own slot reads every value before overwriting it): wait for the tagged
// sources, sum all sources in order, store the elements inside [lo, hi).
template <int DT>
__device__ __forceinline__ void LLReceive(const Task& t, void* const* ptrs, uint64_t begin, uint64_t end,
                                          uint32_t flag, uint64_t parity_off, uint64_t timeout_ns,
                                          int* error_flag) {
  constexpr uint32_t kEs = DT == RS_BF16 ? 2 : 4;
  constexpr int kLLBatch = 8;
  void* const* src = ptrs + t.ptr_begin;
  void* const* dst = src + t.nsrc;
  bool any_result = false;
  for (int j = 0; j < t.ndst; ++j) any_result |= !(reinterpret_cast<uintptr_t>(dst[j]) & 1u);
  if (!any_result) return;
  const char* local = LLLocal(t, src);
  const uint64_t stride = static_cast<uint64_t>(blockDim.x) * 8u;
  // Small pieces with >= 2 remote sources: overlap the sources' latencies
  // (measured K=4 1 KiB AllReduce 9.4 -> 7.9 us); larger pieces keep the
  // 8-deep per-source batches (the wide path was slower from 16 KiB).
  if (t.nsrc >= 3 && t.nsrc <= kLLWide && end - begin <= stride * 4) {
    LLReceiveWide<DT>(t, src, dst, local, begin, end, flag, parity_off, timeout_ns, error_flag);
    return;
  }
  // bf16 keeps only the f32 accumulators and the last source's packets (a
  // single source is then stored raw); the other dtypes accumulate in `out`.
  constexpr bool kF32Acc = DT == RS_BF16;
  for (uint64_t x0 = begin + static_cast<uint64_t>(threadIdx.x) * 8u; x0 < end; x0 += stride * kLLBatch) {
    uint2 mine[kLLBatch], out[kF32Acc ? 1 : kLLBatch], v[kLLBatch];
    float f[kF32Acc ? kLLBatch : 1][4];
#pragma unroll
    for (int b = 0; b < kLLBatch; ++b) {
      const uint64_t x = x0 + b * stride;
      mine[b] = (local && x < end) ? *reinterpret_cast<const uint2*>(local + x) : make_uint2(0, 0);
    }
    // Sum in source order; a single source is a raw copy.
    for (int i = 0; i < t.nsrc; ++i) {
      const uintptr_t s = reinterpret_cast<uintptr_t>(src[i]);
      if (s & 1u) {
        const char* base = reinterpret_cast<const char*>((s & ~uintptr_t{1}) + parity_off);
        uint4 pk[kLLBatch];
#pragma unroll
        for (int b = 0; b < kLLBatch; ++b) {  // all loads in flight at once
          const uint64_t x = x0 + b * stride;
          pk[b] = x < end ? LoadVolatile16(base + 2 * x) : make_uint4(0, flag, 0, flag);
        }
#pragma unroll
        for (int b = 0; b < kLLBatch; ++b) {
          if (pk[b].y != flag || pk[b].w != flag) {
            const uint2 late = LoadLL(base + 2 * (x0 + b * stride), flag, timeout_ns, error_flag);
            pk[b] = make_uint4(late.x, flag, late.y, flag);
          }
          v[b] = make_uint2(pk[b].x, pk[b].z);
        }
      } else {
#pragma unroll
        for (int b = 0; b < kLLBatch; ++b) v[b] = mine[b];
      }
#pragma unroll
      for (int b = 0; b < kLLBatch; ++b) {
        if constexpr (kF32Acc) {
          float g[4];
          BF16Acc::Widen(v[b].x, g[0], g[1]);
          BF16Acc::Widen(v[b].y, g[2], g[3]);
#pragma unroll
          for (int k = 0; k < 4; ++k) f[b][k] = i == 0 ? g[k] : __fadd_rn(f[b][k], g[k]);
        } else {
          out[b] = i == 0 ? v[b] : AddPacket<DT>(out[b], v[b]);
        }
      }
    }
#pragma unroll
    for (int b = 0; b < kLLBatch; ++b) {
      uint2 o;
      if constexpr (kF32Acc) {
        o = t.nsrc > 1 ? make_uint2(BF16Acc::Narrow(f[b][0], f[b][1]), BF16Acc::Narrow(f[b][2], f[b][3])) : v[b];
      } else {
        o = out[b];
      }
      const uint64_t x = x0 + b * stride;
      if (x >= end) continue;
      const bool whole = x >= t.lo && x + 8 <= t.hi;
      for (int j = 0; j < t.ndst; ++j) {
        const uintptr_t d = reinterpret_cast<uintptr_t>(dst[j]);
        if (d & 1u) continue;
        char* base = reinterpret_cast<char*>(d);
        if (whole) {
          *reinterpret_cast<uint2*>(base + x) = o;
          continue;
        }
        // Edge packet: only the elements inside [lo, hi).
        const char* bytes = reinterpret_cast<const char*>(&o);
        for (uint32_t e = 0; e < 8; e += kEs) {
          if (x + e < t.lo || x + e >= t.hi) continue;
          if (kEs == 2) *reinterpret_cast<uint16_t*>(base + x + e) = *reinterpret_cast<const uint16_t*>(bytes + e);
          else *reinterpret_cast<uint32_t*>(base + x + e) = *reinterpret_cast<const uint32_t*>(bytes + e);
        }
      }
    }
  }
}

// Profiling builds only: %globaltimer stamps by thread 0 — per piece p
// trace[3p] = start, [3p+1] = inputs ready (after flag waits), [3p+2] = end;
// per CTA b (after the pieces) trace[3*npieces + 2b] = entry,
// [3*npieces + 2b + 1] = entry barrier passed.
#ifdef RS_PROFILING_AIDS
#define RS_TRACE(idx)                                   \
  do {                                                  \
    if (a.trace && threadIdx.x == 0) a.trace[idx] = GlobalTimer(); \
  } while (0)
#else
#define RS_TRACE(idx) \
  do {                \
  } while (0)
#endif

// One launch phase of one rank: entry barrier, tasks, exit.
// cta / ncta: this CTA's index among the rank's CTAs and their count
// (blockIdx.x / gridDim.x, except in emulated-rank launches).
template <int DT, int kUnroll, bool kLL, bool kNc>
__device__ __forceinline__ void Phase(const StepArgs& a, const uint64_t base, const uint32_t cta,
                                      const uint32_t ncta) {
  // 1. First step of a run: publish "my inputs are in place" to every peer.
  if (a.step == 0 && cta == 0 && threadIdx.x < a.nsignal) {
    // Inputs were written by earlier stream work (complete at kernel
    // boundaries; peers read them through this GPU's L2): no fence needed.
    if (RS_SYNC_STRICT) FenceSys();
    SignalStore(a.signal_ptrs[threadIdx.x], base);
  }
  // 2. Entry barrier: the ranks whose buffers this step touches (and whose
  //    previous-step writers) have finished the previous step.
  RS_TRACE(3ull * a.npieces + 2ull * cta);
  if (threadIdx.x < a.nwait) {
    WaitAtLeast(a.inbox + a.wait_ranks[threadIdx.x], base + a.step - a.wait_lag, a.timeout_ns, a.error_flag);
  }
  __syncthreads();
  RS_TRACE(3ull * a.npieces + 2ull * cta + 1);
  if (a.has_nvls) FenceProxyAlias();

  // 3. Pieces, grid-strided; tasks are ordered by piece_begin. One-shot
  //    phases first push every packet this CTA sends (sweep 1), so each CTA
  //    pays one NVLink round trip however many pieces it walks.
  const uint64_t epoch = base + a.step + 1;
  const uint64_t parity_off = (epoch & 1) * a.ll_parity_stride;
  auto ll_range = [&](const Task& t, uint32_t p, uint64_t& begin, uint64_t& end) {
    begin = (t.lo & ~uint64_t{7}) + static_cast<uint64_t>(p - t.piece_begin) * kLLPieceBytes;
    end = min((t.hi + 7) & ~uint64_t{7}, begin + kLLPieceBytes);
  };
  if constexpr (kLL) {
    uint32_t c = 0;
    for (uint32_t p = cta; p < a.npieces; p += ncta) {
      while (c + 1 < a.ntasks && a.tasks[c + 1].piece_begin <= p) ++c;
      const Task& t = a.tasks[c];
      if (t.mode != kModeLL) continue;
      uint64_t begin, end;
      ll_range(t, p, begin, end);
      LLSend(t, a.ptrs, begin, end, static_cast<uint32_t>(epoch), parity_off);
    }
  }
  uint32_t cur = 0;
  auto run_piece = [&](const uint32_t p) {
    while (cur + 1 < a.ntasks && a.tasks[cur + 1].piece_begin <= p) ++cur;
    const Task& t = a.tasks[cur];
    if (kLL && t.mode == kModeLL) {
      uint64_t begin, end;
      ll_range(t, p, begin, end);
      LLReceive<DT>(t, a.ptrs, begin, end, static_cast<uint32_t>(epoch), parity_off, a.timeout_ns, a.error_flag);
      return;
    }
    RS_TRACE(3ull * p);
    RS_CHECK(t.lo <= t.hi && t.hi <= a.slot_limit, a.error_flag, kCheckRange, t.hi, a.slot_limit);
    RS_CHECK(p >= t.piece_begin && (cur + 1 >= a.ntasks || p < a.tasks[cur + 1].piece_begin), a.error_flag,
             kCheckPiece, p, t.piece_begin);
    if (t.mode == kModeFlagSend || t.mode == kModeFlagRecv) {
      // Push variant, one flag_chunk piece: land it and raise its flag, or
      // wait for every pushed source's flag and reduce it.
      const uint32_t k = p - t.piece_begin;
      const uint64_t chunk = static_cast<uint64_t>(blockDim.x) * kUnroll * 16u;
      void* const* flags = a.ptrs + t.ptr_begin + t.nsrc + t.ndst;
      if (t.mode == kModeFlagRecv) {
        // Reducing pieces are recv_piece bytes (a divisor of flag_chunk), so
        // the reduce work of a mid-size step spreads over every CTA; each
        // waits for the flags of the landing chunk that contains it.
        const uint64_t begin = t.lo + static_cast<uint64_t>(k) * a.recv_piece;
        const uint64_t end = min(t.hi, begin + a.recv_piece);
        const uint64_t fk = (begin - t.lo) / a.flag_chunk;
#ifdef RS_PROFILING_AIDS
        const bool skip_wait = a.solo != 0;
#else
        constexpr bool skip_wait = false;
#endif
        if (threadIdx.x < t.nsrc && flags[threadIdx.x] && !skip_wait) {
          WaitAtLeast(static_cast<const uint64_t*>(flags[threadIdx.x]) + fk, epoch, a.timeout_ns, a.error_flag);
          // a chunk flag of a later run: the sender re-landed this chunk before we reduced it
          RS_CHECK(*reinterpret_cast<const volatile uint64_t*>(static_cast<const uint64_t*>(flags[threadIdx.x]) + fk) <=
                       epoch || Failed(a.error_flag),
                   a.error_flag, kCheckFlagFuture,
                   *reinterpret_cast<const volatile uint64_t*>(static_cast<const uint64_t*>(flags[threadIdx.x]) + fk),
                   epoch);
        }
        __syncthreads();
        RS_TRACE(3ull * p + 1);
        if (a.remote256 && t.nsrc >= 2 && t.nsrc <= 4 && ((t.lo | t.hi) & 31) == 0) {
          const uint64_t wchunk = static_cast<uint64_t>(blockDim.x) * 32u;
          for (uint64_t c = begin; c < end; c += wchunk) WideChunk32<DT, 4, true>(t, a.ptrs, c, min(end, c + wchunk));
        } else if (a.wide_loads && t.nsrc >= 2 && t.nsrc <= 4) {
          constexpr uint64_t kW = 2;
          const uint64_t wchunk = static_cast<uint64_t>(blockDim.x) * kW * 16u;
          for (uint64_t c = begin; c < end; c += wchunk)
            VectorChunkWide<DT, 4, kW, true>(t, a.ptrs, c, min(end, c + wchunk));
        } else if (a.wide_loads && t.nsrc > 4 && t.nsrc <= 8) {
          const uint64_t wchunk = static_cast<uint64_t>(blockDim.x) * 16u;
          for (uint64_t c = begin; c < end; c += wchunk)
            VectorChunkWide<DT, 8, 1, true>(t, a.ptrs, c, min(end, c + wchunk));
        } else {
          for (uint64_t c = begin; c < end; c += chunk)
            VectorChunk<DT, kUnroll, kNc, true>(t, a.ptrs, c, min(end, c + chunk));
        }
      } else {
        const uint64_t begin = t.lo + static_cast<uint64_t>(k) * a.flag_chunk;
        const uint64_t end = min(t.hi, begin + a.flag_chunk);
        if (a.remote256 && t.nsrc == 1 && ((t.lo | t.hi) & 31) == 0) {
          for (uint64_t c = begin; c < end; c += chunk) RemoteCopyChunk32<kUnroll / 2>(t, a.ptrs, c, min(end, c + chunk));
        } else {
          for (uint64_t c = begin; c < end; c += chunk)
            VectorChunk<DT, kUnroll, kNc>(t, a.ptrs, c, min(end, c + chunk));
        }
        __syncthreads();
        RS_TRACE(3ull * p + 1);
        if (threadIdx.x == 0) {
          FenceSys();
          StoreRelaxedSys(static_cast<uint64_t*>(flags[0]) + k, epoch);
        }
      }
      RS_TRACE(3ull * p + 2);
      return;
    }
    if (t.vec) {
      const uint64_t begin = t.lo + static_cast<uint64_t>(p - t.piece_begin) * a.piece_bytes;
      const uint64_t end = min(t.hi, begin + a.piece_bytes);
      const uint64_t chunk = static_cast<uint64_t>(blockDim.x) * kUnroll * 16u;
      bool done = false;
      if constexpr (DT != RS_I32 && !kNc) {  // multicast objects only exist across GPUs
        if (t.mode == kModeNvlsAllReduce) {
          for (uint64_t c = begin; c < end; c += chunk) NvlsChunk<DT, kUnroll>(t, a.ptrs, c, min(end, c + chunk));
          done = true;
        } else if (t.mode == kModeNvlsReduce) {
          for (uint64_t c = begin; c < end; c += chunk)
            NvlsReduceChunk<DT, kUnroll>(t, a.ptrs, c, min(end, c + chunk));
          done = true;
        }
      }
      if constexpr (!kNc) {
        if (t.mode == kModeNvlsBroadcast) {  // a bit copy: every dtype
          for (uint64_t c = begin; c < end; c += chunk) NvlsBroadcastChunk<kUnroll>(t, a.ptrs, c, min(end, c + chunk));
          done = true;
        }
      }
      if constexpr (!kNc) {
        if (!done && a.remote256 && t.nsrc >= 2 && t.nsrc <= 4 && ((t.lo | t.hi) & 31) == 0) {
          const uint64_t wchunk = static_cast<uint64_t>(blockDim.x) * 32u;
          for (uint64_t c = begin; c < end; c += wchunk) WideChunk32<DT, 4>(t, a.ptrs, c, min(end, c + wchunk));
          done = true;
        }
        if (!done && a.wide_loads && t.nsrc >= 2 && t.nsrc <= 8) {
          // cross-GPU sums: every source in flight at once (see VectorChunkWide)
          if (t.nsrc <= 4) {
            constexpr uint64_t kW = 2;
            const uint64_t wchunk = static_cast<uint64_t>(blockDim.x) * kW * 16u;
            for (uint64_t c = begin; c < end; c += wchunk)
              VectorChunkWide<DT, 4, kW>(t, a.ptrs, c, min(end, c + wchunk));
          } else {
            const uint64_t wchunk = static_cast<uint64_t>(blockDim.x) * 16u;
            for (uint64_t c = begin; c < end; c += wchunk)
              VectorChunkWide<DT, 8, 1>(t, a.ptrs, c, min(end, c + wchunk));
          }
          done = true;
        }
      }
      if constexpr (kNc && kUnroll == 8) {  // (unroll 4 + 256-bit: spills, measured -20 %)
        // one GPU, single-source copy with a 32-byte aligned body: 256-bit
        // vectors (kUnroll / 2 per thread, the same bytes in flight)
        if (!done && a.vec256 && ((t.lo | t.hi) & 31) == 0) {
          if (t.nsrc == 1) {
            for (uint64_t c = begin; c < end; c += chunk) CopyChunk32<kUnroll / 2>(t, a.ptrs, c, min(end, c + chunk));
            done = true;
          } else if (a.vec256 >= 2) {
            for (uint64_t c = begin; c < end; c += chunk)
              SumChunk32<DT, kUnroll / 2>(t, a.ptrs, c, min(end, c + chunk));
            done = true;
          }
        }
      }
      if (!done) {
        for (uint64_t c = begin; c < end; c += chunk) VectorChunk<DT, kUnroll, kNc>(t, a.ptrs, c, min(end, c + chunk));
      }
    } else {
      ScalarTask<DT>(t, a.ptrs);
    }
    RS_TRACE(3ull * p + 2);
  };
  // Push phases (a.dynamic == 1): pieces are handed out in launch order
  // through an atomic counter, so a CTA takes a wave's reducing piece only
  // after every landing piece of that wave (and of wave_lag later waves) has
  // been taken (no CTA sits on a flag wait while landing work is left
  // unclaimed; deadlock-free because landing pieces never wait). Other
  // phases: static grid stride (0) or the prefetched queue (2, below).
  __shared__ uint32_t next_piece;
  auto next = [&](uint32_t p) -> uint32_t {
    if (!a.dynamic) return p + ncta;
    if (threadIdx.x == 0) next_piece = atomicAdd(a.piece_counter, 1u);
    __syncthreads();
    const uint32_t q = next_piece;
    __syncthreads();
    return q;
  };
  // a.dynamic == 2 (phases without chunk flags, plan option piece_queue):
  // thread 0 reserves the next piece before working on the current one, so
  // the atomic's round trip hides under the piece. Against the static stride
  // this balances the SMs that see slower HBM (two dies): same DRAM bytes,
  // 1-GPU AllReduce 690 -> 624 us, Broadcast 399 -> 324 us.
  uint32_t p = a.dynamic ? next(0) : cta;
  while (p < a.npieces) {
    uint32_t reserved = 0;
    if (a.dynamic == 2 && threadIdx.x == 0) reserved = atomicAdd(a.piece_counter, 1u);
    run_piece(p);
    if (a.dynamic == 2) {
      if (threadIdx.x == 0) next_piece = reserved;
      __syncthreads();
      p = next_piece;
      __syncthreads();
    } else {
      p = next(p);
    }
  }
  if (a.dynamic && threadIdx.x == 0 && atomicAdd(a.piece_counter + 1, 1u) == ncta - 1) {
    // last CTA out: reset the queue for the next launch on this rank
    atomicExch(a.piece_counter, 0u);
    atomicExch(a.piece_counter + 1, 0u);
  }

  // 4. Exit: the last CTA to finish publishes the step's epoch to all ranks
  //    (skipped when no peer waits for it, e.g. after a one-shot last step).
  const bool last_step = a.step + 1 == a.num_steps;
  const bool publish = a.signal_done && a.nsignal > 0;
  const bool advance = last_step && a.nsignal > 0;
  if (!publish && !advance) return;
  // The CTA barrier orders every thread's stores before thread 0's fence
  // (cumulativity); one fence per CTA instead of one per thread.
  __syncthreads();
  if (threadIdx.x == 0) {
    if (publish) {
      if (a.has_nvls) FenceProxyAlias();
      FenceSys();
    }
    const bool last = ncta == 1 || atomicAdd(a.arrive_counter, 1u) == ncta - 1;
    if (last) {
      if (ncta > 1) atomicExch(a.arrive_counter, 0u);
      if (publish) {
        if (RS_SYNC_STRICT || ncta > 1) FenceSys();  // acquire the other CTAs' releases
        for (uint32_t q = 0; q < a.nsignal; ++q) SignalStore(a.signal_ptrs[q], base + a.step + 1);
      }
      if (last_step) {
        // 5. Last step: the run is complete here only once every rank that
        //    writes into our slots has finished too; then advance the base.
        for (uint32_t i = 0; i < a.nfinal; ++i) {
          WaitAtLeast(a.inbox + a.final_ranks[i], base + a.num_steps, a.timeout_ns, a.error_flag);
        }
        *reinterpret_cast<volatile uint64_t*>(a.epoch_base) = base + a.num_steps + 1;
      }
    }
  }
}

template <int DT, int kUnroll, bool kLL, bool kNc>
__global__ void __launch_bounds__(512, kUnroll == 4 ? 2 : 1) StepKernel(const __grid_constant__ StepArgs a) {
  // Programmatic dependent launch: the next step's grid may be scheduled as
  // soon as this one runs (its launch latency hides under this step), but
  // every step first waits here until the previous grid on the stream has
  // completed and its memory is visible — the same ordering as a plain
  // stream launch. (No-ops for launches without the PDL attribute.)
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // Run base epoch (device resident; advanced by the previous run's last step).
  const uint64_t base = a.nsignal ? *reinterpret_cast<volatile uint64_t*>(a.epoch_base) : 0;
  Phase<DT, kUnroll, kLL, kNc>(a, base, blockIdx.x, gridDim.x);
}

// Emulated ranks (validation on one GPU): every rank's step of one phase in
// ONE cooperative launch, CTAs [prefix[r], prefix[r+1]) acting as rank r's
// grid. Co-residency is what makes ranks that wait on each other safe on a
// single GPU (separate launches are not guaranteed to run concurrently).
template <int DT, int kUnroll, bool kLL>
__global__ void __launch_bounds__(512, 1) EmulatedStepKernel(const __grid_constant__ EmulatedArgs e) {
  asm volatile("griddepcontrol.wait;" ::: "memory");
  uint32_t r = 0;
  while (r + 1 < e.nranks && blockIdx.x >= e.prefix[r + 1]) ++r;
  const StepArgs& a = e.args[r];
  const uint64_t base = a.nsignal ? *reinterpret_cast<volatile uint64_t*>(a.epoch_base) : 0;
  Phase<DT, kUnroll, kLL, false>(a, base, blockIdx.x - e.prefix[r], e.prefix[r + 1] - e.prefix[r]);
}

template <int U>
int Occupancy(int dtype, int threads) {
  int blocks = 0;
  cudaError_t e = cudaSuccess;
  switch (dtype) {
    case RS_F32: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, StepKernel<RS_F32, U, false, false>, threads, 0); break;
    case RS_BF16: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, StepKernel<RS_BF16, U, false, false>, threads, 0); break;
    default: e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, StepKernel<RS_I32, U, false, false>, threads, 0); break;
  }
  if (e != cudaSuccess || blocks < 1) {
    cudaGetLastError();
    return 1;
  }
  return blocks;
}

template <int DT, int U, bool LL, bool NC>
cudaError_t LaunchOne(const StepArgs& a, int grid, int block, cudaStream_t stream, bool pdl) {
  if (!pdl) {
    StepKernel<DT, U, LL, NC><<<grid, block, 0, stream>>>(a);
    return cudaGetLastError();
  }
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(block);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, StepKernel<DT, U, LL, NC>, a);
}

template <int U, bool LL, bool NC>
cudaError_t Launch(const StepArgs& a, int grid, int block, cudaStream_t stream) {
  const bool pdl = a.pdl != 0;
  switch (a.dtype) {
    case RS_F32: return LaunchOne<RS_F32, U, LL, NC>(a, grid, block, stream, pdl);
    case RS_BF16: return LaunchOne<RS_BF16, U, LL, NC>(a, grid, block, stream, pdl);
    case RS_I32: return LaunchOne<RS_I32, U, LL, NC>(a, grid, block, stream, pdl);
    default: return cudaErrorInvalidValue;
  }
}

// NVLS self-check: f32 AllReduce of [lo, hi) through the multicast address
// (the same instructions as the bf16/f32 NVLS tasks) — see EnsureMulticast.
__global__ void NvlsSelfCheckKernel(char* mc, uint64_t lo, uint64_t hi) {
  FenceProxyAlias();
  for (uint64_t off = lo + (static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 16u; off < hi;
       off += static_cast<uint64_t>(gridDim.x) * blockDim.x * 16u) {
    uint4 v;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "l"(mc + off)
                 : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + off), "r"(v.x),
                 "r"(v.y), "r"(v.z), "r"(v.w)
                 : "memory");
  }
  FenceProxyAlias();
  asm volatile("fence.acq_rel.sys;" ::: "memory");
}

template <int DT, int U, bool LL>
cudaError_t LaunchEmulatedOne(const EmulatedArgs& e, int block, cudaStream_t stream) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(e.prefix[e.nranks]);
  cfg.blockDim = dim3(block);
  cfg.stream = stream;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeCooperative;
  attr[0].val.cooperative = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, EmulatedStepKernel<DT, U, LL>, e);
}

template <int U, bool LL>
int EmulatedOccupancy(int dtype, int threads) {
  int blocks = 0;
  cudaError_t err = cudaSuccess;
  switch (dtype) {
    case RS_F32: err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, EmulatedStepKernel<RS_F32, U, LL>, threads, 0); break;
    case RS_BF16: err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, EmulatedStepKernel<RS_BF16, U, LL>, threads, 0); break;
    default: err = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&blocks, EmulatedStepKernel<RS_I32, U, LL>, threads, 0); break;
  }
  if (err != cudaSuccess || blocks < 1) {
    cudaGetLastError();
    return 1;
  }
  return blocks;
}

}  // namespace

cudaError_t LaunchEmulated(const EmulatedArgs& e, bool ll, int block, cudaStream_t stream) {
  switch (e.args[0].dtype) {
    case RS_F32: return ll ? LaunchEmulatedOne<RS_F32, 2, true>(e, block, stream) : LaunchEmulatedOne<RS_F32, 4, false>(e, block, stream);
    case RS_BF16: return ll ? LaunchEmulatedOne<RS_BF16, 2, true>(e, block, stream) : LaunchEmulatedOne<RS_BF16, 4, false>(e, block, stream);
    case RS_I32: return ll ? LaunchEmulatedOne<RS_I32, 2, true>(e, block, stream) : LaunchEmulatedOne<RS_I32, 4, false>(e, block, stream);
    default: return cudaErrorInvalidValue;
  }
}

int EmulatedResidentCtas(int dtype, int threads, bool ll) {
  return ll ? EmulatedOccupancy<2, true>(dtype, threads) : EmulatedOccupancy<4, false>(dtype, threads);
}

cudaError_t LaunchNvlsSelfCheck(char* mc, uint64_t lo, uint64_t hi, cudaStream_t stream) {
  NvlsSelfCheckKernel<<<8, 256, 0, stream>>>(mc, lo, hi);
  return cudaGetLastError();
}

int MaxResidentCtas(int dtype, int threads, int unroll) {
  return unroll == 8 ? Occupancy<8>(dtype, threads) : Occupancy<4>(dtype, threads);
}

cudaError_t LaunchStep(const StepArgs& args, int grid, int block, int unroll, cudaStream_t stream) {
  // One-shot phases only exist across GPUs (never .nc); (512, 1): 128 registers.
  if (args.has_ll) return Launch<2, true, false>(args, grid, block, stream);
  if (args.local_only) {
    return unroll == 8 ? Launch<8, false, true>(args, grid, block, stream)
                       : Launch<4, false, true>(args, grid, block, stream);
  }
  return unroll == 8 ? Launch<8, false, false>(args, grid, block, stream)
                     : Launch<4, false, false>(args, grid, block, stream);
}

}  // namespace rs
