// HBM write-path probe (one GPU): how fast can SM stores write HBM, and what
// does a 1-read / k-write copy (the local Broadcast / AllGather step shape)
// reach with different store forms? Non-zero data everywhere (no help from
// zero-value paths). Prints GB/s of algorithmic bytes (reads + writes).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/hbm_write_probe tools/hbm_write_probe.cu
//   ./tools/hbm_write_probe [MiB per buffer]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) {                                                                 \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__);   \
      std::exit(1);                                                                          \
    }                                                                                        \
  } while (0)

enum Store { kPlain = 0, kNoAlloc = 1, kCs = 2, kEvictFirst = 3, kWb = 4 };

// 256-bit (sm_100) load / store: 32 bytes per thread per instruction.
struct V8 {
  uint32_t r[8];
};
template <int S>
__device__ __forceinline__ void St8(void* p, const V8& v) {
  if constexpr (S == kEvictFirst) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p),
                 "r"(v.r[0]), "r"(v.r[1]), "r"(v.r[2]), "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]),
                 "r"(v.r[7]) : "memory");
  } else {
    asm volatile("st.global.L1::no_allocate.v8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};" ::"l"(p), "r"(v.r[0]),
                 "r"(v.r[1]), "r"(v.r[2]), "r"(v.r[3]), "r"(v.r[4]), "r"(v.r[5]), "r"(v.r[6]), "r"(v.r[7]) : "memory");
  }
}
__device__ __forceinline__ V8 Ld8(const void* p) {
  V8 v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=r"(v.r[0]), "=r"(v.r[1]), "=r"(v.r[2]), "=r"(v.r[3]), "=r"(v.r[4]), "=r"(v.r[5]), "=r"(v.r[6]),
                 "=r"(v.r[7])
               : "l"(p));
  return v;
}

template <int S, int U>
__global__ void fill8_kernel(V8* dst, size_t n, uint32_t seed) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n; base += stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + static_cast<size_t>(u) * blockDim.x;
      V8 v;
#pragma unroll
      for (int k = 0; k < 8; ++k) v.r[k] = seed ^ static_cast<uint32_t>(i * 8 + k);
      if (i < n) St8<S>(dst + i, v);
    }
  }
}

template <int S, int U, int K>
__global__ void bcast8_kernel(V8* const* dst, const V8* src, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n; base += stride) {
    V8 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + static_cast<size_t>(u) * blockDim.x;
      if (i < n) v[u] = Ld8(src + i);
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + static_cast<size_t>(u) * blockDim.x;
        if (i < n) St8<S>(dst[k] + i, v[u]);
      }
    }
  }
}

template <int S>
__device__ __forceinline__ void St(void* p, const uint4& v) {
  if constexpr (S == kPlain) {
    asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  } else if constexpr (S == kNoAlloc) {
    asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z),
                 "r"(v.w) : "memory");
  } else if constexpr (S == kCs) {
    asm volatile("st.global.cs.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  } else if constexpr (S == kEvictFirst) {
    asm volatile("st.global.L1::no_allocate.L2::evict_first.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
                 "r"(v.z), "r"(v.w) : "memory");  // (ptxas: evict_first needs 256-bit stores; kept for kWide256)
  } else {
    asm volatile("st.global.wb.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
  }
}

// write-only fill: U vectors per thread per iteration, grid-stride
template <int S, int U>
__global__ void fill_kernel(uint4* dst, size_t n, uint32_t seed) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n; base += stride) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + static_cast<size_t>(u) * blockDim.x;
      if (i < n) St<S>(dst + i, make_uint4(seed ^ static_cast<uint32_t>(i), seed, ~static_cast<uint32_t>(i), 7u));
    }
  }
}

// 1 read, K writes (the local Broadcast shape), U vectors per thread in flight
template <int S, int U, int K>
__global__ void bcast_kernel(uint4* const* dst, const uint4* src, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n; base += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + static_cast<size_t>(u) * blockDim.x;
      if (i < n)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(src + i));
    }
#pragma unroll
    for (int k = 0; k < K; ++k) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + static_cast<size_t>(u) * blockDim.x;
        if (i < n) St<S>(dst[k] + i, v[u]);
      }
    }
  }
}

template <typename F>
double Time(F f, int iters) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  f();
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int i = 0; i < iters; ++i) {
    CK(cudaEventRecord(a));
    f();
    CK(cudaEventRecord(b));
    CK(cudaEventSynchronize(b));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, a, b));
    if (ms < best) best = ms;
  }
  return best * 1e-3;
}

template <int S, int U>
void RunFill(const char* name, uint4* d, size_t n, int grid, int block) {
  const double s = Time([&] { fill_kernel<S, U><<<grid, block>>>(d, n, 0x9e3779b9u); }, 10);
  std::printf("{\"probe\": \"fill %s U=%d grid=%d block=%d\", \"GBps\": %.1f}\n", name, U, grid, block,
              n * 16.0 / s / 1e9);
}

template <int S, int U, int K>
void RunBcast(const char* name, uint4* const* dptrs, const uint4* src, size_t n, int grid, int block) {
  const double s = Time([&] { bcast_kernel<S, U, K><<<grid, block>>>(dptrs, src, n); }, 10);
  std::printf("{\"probe\": \"1r%dw %s U=%d grid=%d block=%d\", \"GBps\": %.1f}\n", K, name, U, grid, block,
              n * 16.0 * (1 + K) / s / 1e9);
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? std::strtoull(argv[1], nullptr, 10) : 256;
  const size_t bytes = mib << 20, n = bytes / 16;
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  uint4* buf[8];
  for (auto& p : buf) CK(cudaMalloc(&p, bytes));
  uint4** dptrs = nullptr;
  CK(cudaMalloc(&dptrs, sizeof(buf)));
  CK(cudaMemcpy(dptrs, buf + 1, 7 * sizeof(uint4*), cudaMemcpyHostToDevice));
  fill_kernel<kPlain, 4><<<sms * 4, 512>>>(buf[0], n, 12345u);
  CK(cudaDeviceSynchronize());
  {
    const double s = Time([&] { CK(cudaMemsetAsync(buf[7], 0x5a, bytes)); }, 10);
    std::printf("{\"probe\": \"cudaMemsetAsync 0x5a\", \"GBps\": %.1f}\n", bytes / s / 1e9);
  }
  RunFill<kPlain, 4>("plain", buf[7], n, sms * 4, 512);
  RunFill<kNoAlloc, 4>("L1::no_allocate", buf[7], n, sms * 4, 512);
  RunFill<kCs, 4>("cs", buf[7], n, sms * 4, 512);
  {
    const size_t n8 = bytes / 32;
    V8* d8 = reinterpret_cast<V8*>(buf[7]);
    double t = Time([&] { fill8_kernel<kNoAlloc, 4><<<sms * 4, 512>>>(d8, n8, 7u); }, 10);
    std::printf("{\"probe\": \"fill 256-bit no_allocate U=4\", \"GBps\": %.1f}\n", bytes / t / 1e9);
    t = Time([&] { fill8_kernel<kEvictFirst, 4><<<sms * 4, 512>>>(d8, n8, 7u); }, 10);
    std::printf("{\"probe\": \"fill 256-bit evict_first U=4\", \"GBps\": %.1f}\n", bytes / t / 1e9);
    t = Time([&] { fill8_kernel<kNoAlloc, 2><<<sms * 8, 256>>>(d8, n8, 7u); }, 10);
    std::printf("{\"probe\": \"fill 256-bit no_allocate U=2 256thr\", \"GBps\": %.1f}\n", bytes / t / 1e9);
    V8* const* dp8 = reinterpret_cast<V8* const*>(dptrs);
    const V8* s8 = reinterpret_cast<const V8*>(buf[0]);
    t = Time([&] { bcast8_kernel<kNoAlloc, 4, 3><<<sms, 512>>>(dp8, s8, n8); }, 10);
    std::printf("{\"probe\": \"1r3w 256-bit no_allocate U=4\", \"GBps\": %.1f}\n", bytes * 4.0 / t / 1e9);
    t = Time([&] { bcast8_kernel<kEvictFirst, 4, 3><<<sms, 512>>>(dp8, s8, n8); }, 10);
    std::printf("{\"probe\": \"1r3w 256-bit evict_first U=4\", \"GBps\": %.1f}\n", bytes * 4.0 / t / 1e9);
    t = Time([&] { bcast8_kernel<kNoAlloc, 2, 3><<<sms * 2, 512>>>(dp8, s8, n8); }, 10);
    std::printf("{\"probe\": \"1r3w 256-bit no_allocate U=2 2cta\", \"GBps\": %.1f}\n", bytes * 4.0 / t / 1e9);
    t = Time([&] { bcast8_kernel<kNoAlloc, 4, 7><<<sms, 512>>>(dp8, s8, n8); }, 10);
    std::printf("{\"probe\": \"1r7w 256-bit no_allocate U=4\", \"GBps\": %.1f}\n", bytes * 8.0 / t / 1e9);
    t = Time([&] { bcast8_kernel<kNoAlloc, 4, 1><<<sms, 512>>>(dp8, s8, n8); }, 10);
    std::printf("{\"probe\": \"1r1w 256-bit no_allocate U=4\", \"GBps\": %.1f}\n", bytes * 2.0 / t / 1e9);
  }
  RunFill<kNoAlloc, 8>("L1::no_allocate", buf[7], n, sms * 2, 512);
  RunFill<kNoAlloc, 4>("L1::no_allocate", buf[7], n, sms * 16, 256);
  RunFill<kNoAlloc, 1>("L1::no_allocate", buf[7], n, sms * 32, 256);
  RunBcast<kNoAlloc, 8, 1>("L1::no_allocate", dptrs, buf[0], n, sms, 512);
  RunBcast<kNoAlloc, 8, 3>("L1::no_allocate", dptrs, buf[0], n, sms, 512);
  RunBcast<kNoAlloc, 4, 3>("L1::no_allocate", dptrs, buf[0], n, sms * 2, 512);
  RunBcast<kNoAlloc, 2, 3>("L1::no_allocate", dptrs, buf[0], n, sms * 4, 512);
  RunBcast<kCs, 8, 3>("cs", dptrs, buf[0], n, sms, 512);
  RunBcast<kPlain, 8, 3>("plain", dptrs, buf[0], n, sms, 512);
  RunBcast<kNoAlloc, 8, 7>("L1::no_allocate", dptrs, buf[0], n, sms, 512);
  RunBcast<kNoAlloc, 2, 7>("L1::no_allocate", dptrs, buf[0], n, sms * 4, 512);
  return 0;
}
