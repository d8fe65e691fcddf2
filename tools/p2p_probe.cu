// NVLink / NVSwitch calibration probe (2+ GPUs, one process, peer access).
// Measures what SM-driven peer loads/stores and the copy engines reach on
// this box, per direction, uni- and bidirectional, so the executor's
// roofline denominators are measured rather than assumed.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o p2p_probe tools/p2p_probe.cu
//   ./p2p_probe [MiB]
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CK(x)                                                                        \
  do {                                                                               \
    cudaError_t e_ = (x);                                                            \
    if (e_ != cudaSuccess) {                                                         \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                                  \
    }                                                                                \
  } while (0)

template <int U>
__global__ void copy_kernel(uint4* __restrict__ dst, const uint4* __restrict__ src, size_t n) {
  const size_t stride = static_cast<size_t>(gridDim.x) * blockDim.x * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; base < n;
       base += stride) {
    uint4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + static_cast<size_t>(u) * blockDim.x;
      if (i < n) {
        asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                     : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                     : "l"(src + i));
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      size_t i = base + static_cast<size_t>(u) * blockDim.x;
      if (i < n) dst[i] = v[u];
    }
  }
}

// Bulk-copy (TMA engine) copy: one elected thread per CTA streams chunks
// global -> shared (cp.async.bulk + mbarrier) -> global (cp.async.bulk store),
// kStages chunks in flight.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

template <int kStages>
__global__ void tma_copy_kernel(char* __restrict__ dst, const char* __restrict__ src, size_t bytes,
                                uint32_t chunk) {
  extern __shared__ __align__(128) char smem[];
  __shared__ __align__(8) uint64_t bar[kStages];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < kStages; ++s)
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar[s])));
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const size_t nchunks = (bytes + chunk - 1) / chunk;
  uint32_t phase[kStages] = {};
  auto issue_load = [&](size_t c, int s) {
    const size_t off = c * chunk;
    const uint32_t len = static_cast<uint32_t>(bytes - off < chunk ? bytes - off : chunk);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar[s])), "r"(len)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            smem_u32(smem + static_cast<size_t>(s) * chunk)),
        "l"(src + off), "r"(len), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  size_t k = 0;
  size_t first = blockIdx.x;
  for (int s = 0; s < kStages; ++s) {
    const size_t c = first + static_cast<size_t>(s) * gridDim.x;
    if (c < nchunks) issue_load(c, s);
  }
  for (size_t c = first; c < nchunks; c += gridDim.x, ++k) {
    const int s = static_cast<int>(k % kStages);
    // wait for the load
    uint32_t done = 0;
    while (!done) {
      asm volatile(
          "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
          : "=r"(done)
          : "r"(smem_u32(&bar[s])), "r"(phase[s])
          : "memory");
    }
    phase[s] ^= 1;
    const size_t off = c * chunk;
    const uint32_t len = static_cast<uint32_t>(bytes - off < chunk ? bytes - off : chunk);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst + off),
                 "r"(smem_u32(smem + static_cast<size_t>(s) * chunk)), "r"(len)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    const size_t next = c + static_cast<size_t>(kStages) * gridDim.x;
    if (next < nchunks) issue_load(next, s);
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

struct Buf {
  int dev;
  uint4* a;
  uint4* b;
  cudaStream_t s;
  cudaEvent_t e0, e1;
};

template <int U>
void launch(const Buf& x, uint4* dst, const uint4* src, size_t n, int ctas, int threads) {
  CK(cudaSetDevice(x.dev));
  copy_kernel<U><<<ctas, threads, 0, x.s>>>(dst, src, n);
}

int main(int argc, char** argv) {
  const size_t mib = argc > 1 ? std::atoll(argv[1]) : 512;
  const size_t bytes = mib << 20;
  const size_t n = bytes / 16;
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < 2) {
    std::printf("need 2 GPUs\n");
    return 0;
  }
  std::vector<Buf> g(2);
  for (int d = 0; d < 2; ++d) {
    g[d].dev = d;
    CK(cudaSetDevice(d));
    CK(cudaMalloc(&g[d].a, bytes));
    CK(cudaMalloc(&g[d].b, bytes));
    CK(cudaMemset(g[d].a, 1, bytes));
    CK(cudaMemset(g[d].b, 2, bytes));
    CK(cudaStreamCreateWithFlags(&g[d].s, cudaStreamNonBlocking));
    CK(cudaEventCreate(&g[d].e0));
    CK(cudaEventCreate(&g[d].e1));
    cudaError_t e = cudaDeviceEnablePeerAccess(1 - d, 0);
    if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
    cudaGetLastError();
  }
  auto run = [&](const char* name, bool both, auto body) {
    for (int it = 0; it < 3; ++it) {  // warm-up
      for (int d = 0; d < (both ? 2 : 1); ++d) body(d);
    }
    for (int d = 0; d < 2; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
    }
    const int reps = 5;
    for (int d = 0; d < (both ? 2 : 1); ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(g[d].e0, g[d].s));
    }
    for (int r = 0; r < reps; ++r)
      for (int d = 0; d < (both ? 2 : 1); ++d) body(d);
    float worst = 0;
    for (int d = 0; d < (both ? 2 : 1); ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(g[d].e1, g[d].s));
      CK(cudaEventSynchronize(g[d].e1));
      float ms = 0;
      CK(cudaEventElapsedTime(&ms, g[d].e0, g[d].e1));
      worst = ms > worst ? ms : worst;
    }
    std::printf("%-58s %8.1f GB/s per direction\n", name, bytes * reps / (worst * 1e-3) / 1e9);
  };
  for (int threads : {512, 1024}) {
    for (int ctas_per_sm : {1, 2, 4}) {
      const int ctas = 148 * ctas_per_sm * (threads == 1024 ? 1 : 1);
      if (threads * ctas_per_sm > 2048) continue;
      char name[128];
      std::snprintf(name, sizeof name, "pull 1-dir  (read peer, write local) t=%d ctas=%d U=4", threads, ctas);
      run(name, false, [&](int d) { launch<4>(g[d], g[d].b, g[1 - d].a, n, ctas, threads); });
      std::snprintf(name, sizeof name, "pull 2-dir                          t=%d ctas=%d U=4", threads, ctas);
      run(name, true, [&](int d) { launch<4>(g[d], g[d].b, g[1 - d].a, n, ctas, threads); });
      std::snprintf(name, sizeof name, "push 1-dir  (read local, write peer) t=%d ctas=%d U=4", threads, ctas);
      run(name, false, [&](int d) { launch<4>(g[d], g[1 - d].b, g[d].a, n, ctas, threads); });
      std::snprintf(name, sizeof name, "push 2-dir                          t=%d ctas=%d U=4", threads, ctas);
      run(name, true, [&](int d) { launch<4>(g[d], g[1 - d].b, g[d].a, n, ctas, threads); });
      std::snprintf(name, sizeof name, "pull 2-dir                          t=%d ctas=%d U=8", threads, ctas);
      run(name, true, [&](int d) { launch<8>(g[d], g[d].b, g[1 - d].a, n, ctas, threads); });
      std::snprintf(name, sizeof name, "push 2-dir                          t=%d ctas=%d U=8", threads, ctas);
      run(name, true, [&](int d) { launch<8>(g[d], g[1 - d].b, g[d].a, n, ctas, threads); });
    }
  }
  for (int stages : {4}) {
    for (uint32_t chunk : {16384u, 32768u, 49152u}) {
      const size_t smem_bytes = static_cast<size_t>(stages) * chunk;
      for (int d = 0; d < 2; ++d) {
        CK(cudaSetDevice(d));
        CK(cudaFuncSetAttribute(tma_copy_kernel<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                static_cast<int>(smem_bytes)));
      }
      for (int ctas : {148, 296}) {
        if (smem_bytes * (ctas / 148) > 220 * 1024) continue;
        char name[128];
        auto tma = [&](int d, char* dst, const char* src) {
          CK(cudaSetDevice(d));
          tma_copy_kernel<4><<<ctas, 32, smem_bytes, g[d].s>>>(dst, src, bytes, chunk);
        };
        std::snprintf(name, sizeof name, "tma pull 1-dir chunk=%u ctas=%d", chunk, ctas);
        run(name, false, [&](int d) { tma(d, (char*)g[d].b, (const char*)g[1 - d].a); });
        std::snprintf(name, sizeof name, "tma pull 2-dir chunk=%u ctas=%d", chunk, ctas);
        run(name, true, [&](int d) { tma(d, (char*)g[d].b, (const char*)g[1 - d].a); });
        std::snprintf(name, sizeof name, "tma push 1-dir chunk=%u ctas=%d", chunk, ctas);
        run(name, false, [&](int d) { tma(d, (char*)g[1 - d].b, (const char*)g[d].a); });
        std::snprintf(name, sizeof name, "tma push 2-dir chunk=%u ctas=%d", chunk, ctas);
        run(name, true, [&](int d) { tma(d, (char*)g[1 - d].b, (const char*)g[d].a); });
      }
    }
  }
  run("cudaMemcpyPeerAsync 1-dir", false, [&](int d) {
    CK(cudaSetDevice(d));
    CK(cudaMemcpyPeerAsync(g[1 - d].b, 1 - d, g[d].a, d, bytes, g[d].s));
  });
  run("cudaMemcpyPeerAsync 2-dir", true, [&](int d) {
    CK(cudaSetDevice(d));
    CK(cudaMemcpyPeerAsync(g[1 - d].b, 1 - d, g[d].a, d, bytes, g[d].s));
  });
  run("local HBM copy (d2d)", false, [&](int d) { launch<4>(g[d], g[d].b, g[d].a, n, 296, 512); });
  return 0;
}
