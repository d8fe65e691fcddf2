// NVLS (NVLink SHARP / multimem) feasibility + bandwidth probe, one process
// driving n GPUs. Builds one multicast object over n GPUs, binds a
// cuMemCreate'd buffer of each, and times an AllReduce where GPU i reduces
// its 1/n slice with multimem.ld_reduce and writes it back with multimem.st
// (both through NVSwitch). Reports bus GB/s (2(n-1)/n * D / t).
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o nvls_probe tools/nvls_probe.cu -lcuda
//   ./nvls_probe [n] [MiB]
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <vector>

#define CU(x)                                                                     \
  do {                                                                            \
    CUresult r_ = (x);                                                            \
    if (r_ != CUDA_SUCCESS) {                                                     \
      const char* s_ = nullptr;                                                   \
      cuGetErrorString(r_, &s_);                                                  \
      std::printf("CU error %d (%s) at %s:%d: %s\n", r_, s_ ? s_ : "?", __FILE__, __LINE__, #x); \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)
#define CK(x)                                                                     \
  do {                                                                            \
    cudaError_t e_ = (x);                                                         \
    if (e_ != cudaSuccess) {                                                      \
      std::printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e_), __FILE__, __LINE__); \
      std::exit(1);                                                               \
    }                                                                             \
  } while (0)

__global__ void nvls_allreduce_f32(float* mc, size_t begin, size_t end) {
  for (size_t i = begin + (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < end;
       i += static_cast<size_t>(gridDim.x) * blockDim.x * 4) {
    float a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.v4.f32 {%0, %1, %2, %3}, [%4];"
                 : "=f"(a), "=f"(b), "=f"(c), "=f"(d)
                 : "l"(mc + i)
                 : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "f"(a), "f"(b),
                 "f"(c), "f"(d)
                 : "memory");
  }
}

template <int U>
__global__ void nvls_allreduce_bf16_u(uint32_t* mc, size_t begin, size_t end) {
  const size_t step = static_cast<size_t>(gridDim.x) * blockDim.x * 4 * U;
  for (size_t base = begin + (static_cast<size_t>(blockIdx.x) * blockDim.x * U + threadIdx.x) * 4; base < end;
       base += step) {
    uint32_t v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + static_cast<size_t>(u) * blockDim.x * 4;
      if (i < end)
        asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                     : "=r"(v[u][0]), "=r"(v[u][1]), "=r"(v[u][2]), "=r"(v[u][3])
                     : "l"(mc + i)
                     : "memory");
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + static_cast<size_t>(u) * blockDim.x * 4;
      if (i < end)
        asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(mc + i),
                     "r"(v[u][0]), "r"(v[u][1]), "r"(v[u][2]), "r"(v[u][3])
                     : "memory");
    }
  }
}

__global__ void nvls_allreduce_bf16(uint32_t* mc, size_t begin, size_t end) {
  // indices in 32-bit words (bf16x2)
  for (size_t i = begin + (static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < end;
       i += static_cast<size_t>(gridDim.x) * blockDim.x * 4) {
    uint32_t a, b, c, d;
    asm volatile("multimem.ld_reduce.relaxed.sys.global.add.acc::f32.v4.bf16x2 {%0, %1, %2, %3}, [%4];"
                 : "=r"(a), "=r"(b), "=r"(c), "=r"(d)
                 : "l"(mc + i)
                 : "memory");
    asm volatile("multimem.st.relaxed.sys.global.v4.bf16x2 [%0], {%1, %2, %3, %4};" ::"l"(mc + i), "r"(a), "r"(b),
                 "r"(c), "r"(d)
                 : "memory");
  }
}

int main(int argc, char** argv) {
  int n = argc > 1 ? std::atoi(argv[1]) : 2;
  const size_t mib = argc > 2 ? std::atoll(argv[2]) : 256;
  CU(cuInit(0));
  int ndev = 0;
  CK(cudaGetDeviceCount(&ndev));
  if (ndev < n) {
    std::printf("need %d GPUs, have %d\n", n, ndev);
    return 0;
  }
  for (int d = 0; d < n; ++d) {
    CUdevice dev;
    CU(cuDeviceGet(&dev, d));
    int mc = 0;
    CU(cuDeviceGetAttribute(&mc, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev));
    std::printf("device %d multicast supported: %d\n", d, mc);
    if (!mc) return 0;
  }
  CUmulticastObjectProp prop = {};
  prop.numDevices = n;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t gran = 0;
  prop.size = mib << 20;
  CU(cuMulticastGetGranularity(&gran, &prop, CU_MULTICAST_GRANULARITY_RECOMMENDED));
  size_t bytes = ((mib << 20) + gran - 1) / gran * gran;
  prop.size = bytes;
  std::printf("multicast granularity %zu, size %zu\n", gran, bytes);
  CUmemGenericAllocationHandle mc;
  CU(cuMulticastCreate(&mc, &prop));
  std::vector<CUdevice> devs(n);
  for (int d = 0; d < n; ++d) {
    CU(cuDeviceGet(&devs[d], d));
    CU(cuMulticastAddDevice(mc, devs[d]));
  }
  std::vector<CUdeviceptr> uc(n), mcp(n);
  std::vector<cudaStream_t> streams(n);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaFree(0));
    CUmemAllocationProp ap = {};
    ap.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    ap.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    ap.location.id = d;
    ap.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
    size_t agran = 0;
    CU(cuMemGetAllocationGranularity(&agran, &ap, CU_MEM_ALLOC_GRANULARITY_RECOMMENDED));
    CUmemGenericAllocationHandle phys;
    CU(cuMemCreate(&phys, bytes, &ap, 0));
    CU(cuMulticastBindMem(mc, 0, phys, 0, bytes, 0));
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = d;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    CU(cuMemAddressReserve(&uc[d], bytes, gran, 0, 0));
    CU(cuMemMap(uc[d], bytes, 0, phys, 0));
    CU(cuMemSetAccess(uc[d], bytes, &acc, 1));
    CU(cuMemAddressReserve(&mcp[d], bytes, gran, 0, 0));
    CU(cuMemMap(mcp[d], bytes, 0, mc, 0));
    CU(cuMemSetAccess(mcp[d], bytes, &acc, 1));
    CK(cudaMemset(reinterpret_cast<void*>(uc[d]), 0, bytes));
    CK(cudaStreamCreateWithFlags(&streams[d], cudaStreamNonBlocking));
  }
  // correctness: f32 ones on every GPU -> n after one AllReduce
  const size_t nf = bytes / 4;
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    std::vector<float> ones(1 << 20, 1.0f);
    for (size_t off = 0; off < nf; off += ones.size())
      CK(cudaMemcpy(reinterpret_cast<float*>(uc[d]) + off, ones.data(), 4 * std::min(ones.size(), nf - off),
                    cudaMemcpyHostToDevice));
  }
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  int variant = 0, ctas = 296;
  auto run = [&](bool bf16) {
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      size_t words = bytes / 4;
      size_t per = (words / n + 3) / 4 * 4;
      size_t b = d * per, e = std::min(words, b + per);
      uint32_t* w = reinterpret_cast<uint32_t*>(mcp[d]);
      if (!bf16)
        nvls_allreduce_f32<<<ctas, 512, 0, streams[d]>>>(reinterpret_cast<float*>(mcp[d]), b, e);
      else if (variant == 0)
        nvls_allreduce_bf16<<<ctas, 512, 0, streams[d]>>>(w, b, e);
      else if (variant == 2)
        nvls_allreduce_bf16_u<2><<<ctas, 512, 0, streams[d]>>>(w, b, e);
      else
        nvls_allreduce_bf16_u<4><<<ctas, 512, 0, streams[d]>>>(w, b, e);
    }
  };
  run(false);
  for (int d = 0; d < n; ++d) {
    CK(cudaSetDevice(d));
    CK(cudaDeviceSynchronize());
  }
  for (int d = 0; d < n; ++d) {
    float x[4];
    CK(cudaSetDevice(d));
    CK(cudaMemcpy(x, reinterpret_cast<float*>(uc[d]) + nf / 2, 16, cudaMemcpyDeviceToHost));
    std::printf("device %d value after one AllReduce: %g (expect %d)\n", d, x[0], n);
  }
  {
    size_t mg = 0;
    CU(cuMulticastGetGranularity(&mg, &prop, CU_MULTICAST_GRANULARITY_MINIMUM));
    std::printf("multicast minimum granularity %zu\n", mg);
    CUmemAllocationProp fp = {};
    fp.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    fp.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    fp.location.id = 0;
    fp.requestedHandleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    CUmemGenericAllocationHandle fh;
    CUresult fr = cuMemCreate(&fh, 2 << 20, &fp, 0);
    std::printf("fabric-handle cuMemCreate: %d\n", static_cast<int>(fr));
    if (fr == CUDA_SUCCESS) {
      CUmemFabricHandle exported;
      CUresult er = cuMemExportToShareableHandle(&exported, fh, CU_MEM_HANDLE_TYPE_FABRIC, 0);
      std::printf("fabric-handle export: %d\n", static_cast<int>(er));
    }
    CUmulticastObjectProp fprop = prop;
    fprop.handleTypes = CU_MEM_HANDLE_TYPE_FABRIC;
    fprop.size = mg;
    CUmemGenericAllocationHandle fmc;
    std::printf("fabric-handle cuMulticastCreate: %d\n", static_cast<int>(cuMulticastCreate(&fmc, &fprop)));
  }
  const int cta_opts[] = {148, 296, 592};
  for (int combo = 0; combo < 1 + 3 * 3; ++combo) {
    const int bf = combo > 0;
    if (bf) {
      variant = (combo - 1) / 3 == 0 ? 0 : ((combo - 1) / 3 == 1 ? 2 : 4);
      ctas = cta_opts[(combo - 1) % 3];
    }
    for (int it = 0; it < 3; ++it) run(bf);
    std::vector<cudaEvent_t> e0(n), e1(n);
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaDeviceSynchronize());
      CK(cudaEventCreate(&e0[d]));
      CK(cudaEventCreate(&e1[d]));
      CK(cudaEventRecord(e0[d], streams[d]));
    }
    const int reps = 10;
    for (int r = 0; r < reps; ++r) run(bf);
    float worst = 0;
    for (int d = 0; d < n; ++d) {
      CK(cudaSetDevice(d));
      CK(cudaEventRecord(e1[d], streams[d]));
      CK(cudaEventSynchronize(e1[d]));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0[d], e1[d]));
      worst = std::max(worst, ms);
    }
    const double t = worst / reps * 1e-3;
    std::printf("NVLS AllReduce %s unroll=%d ctas=%d n=%d D=%zu MiB: %.1f us, busbw %.1f GB/s\n",
                bf ? "bf16" : "f32", bf ? (variant ? variant : 1) : 1, ctas, n, bytes >> 20, t * 1e6,
                bytes * 2.0 * (n - 1) / n / t / 1e9);
  }
  return 0;
}
