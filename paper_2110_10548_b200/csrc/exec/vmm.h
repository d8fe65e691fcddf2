// CUDA virtual-memory-management helpers: heaps that can be shared across
// processes as POSIX file descriptors (pidfd_getfd) and bound to NVLink
// multicast (NVLS) objects.
#ifndef REDSYNTH_B200_EXEC_VMM_H_
#define REDSYNTH_B200_EXEC_VMM_H_

#include <cuda.h>

#include <cstdint>
#include <vector>

#include "absl/status/status.h"

// Driver-API entry points resolved at run time through the CUDA runtime
// (cudaGetDriverEntryPoint), so the library never links libcuda: it still
// loads on a machine without a GPU driver (CPU tests, build containers).
namespace rs::drv {
void* Resolve(const char* name);
#define RS_DRV_FN(name)                                                 \
  template <typename... A>                                              \
  inline CUresult name(A... args) {                                     \
    using F = decltype(&::name);                                        \
    static F f = reinterpret_cast<F>(Resolve(#name));                   \
    return f ? f(args...) : CUDA_ERROR_NOT_INITIALIZED;                 \
  }
RS_DRV_FN(cuInit)
RS_DRV_FN(cuGetErrorString)
RS_DRV_FN(cuDeviceGet)
RS_DRV_FN(cuDeviceGetAttribute)
RS_DRV_FN(cuMemCreate)
RS_DRV_FN(cuMemRelease)
RS_DRV_FN(cuMemAddressReserve)
RS_DRV_FN(cuMemAddressFree)
RS_DRV_FN(cuMemMap)
RS_DRV_FN(cuMemUnmap)
RS_DRV_FN(cuMemSetAccess)
RS_DRV_FN(cuMemGetAllocationGranularity)
RS_DRV_FN(cuMemExportToShareableHandle)
RS_DRV_FN(cuMemImportFromShareableHandle)
RS_DRV_FN(cuMulticastCreate)
RS_DRV_FN(cuMulticastAddDevice)
RS_DRV_FN(cuMulticastBindMem)
RS_DRV_FN(cuMulticastUnbind)
RS_DRV_FN(cuMulticastGetGranularity)
#undef RS_DRV_FN
}  // namespace rs::drv

namespace rs {

struct VmmBlock {
  CUmemGenericAllocationHandle handle = 0;
  CUdeviceptr va = 0;
  size_t bytes = 0;
  bool mapped = false;
};

// What a peer needs to import a heap: process id + fd number in that process.
struct VmmShare {
  uint32_t magic;
  int32_t pid;
  int32_t fd;
  uint32_t pad;
  uint64_t bytes;
};
constexpr uint32_t kVmmMagic = 0x31565352u;  // "RSV1"

absl::Status CuStatus(CUresult r, const char* what);

size_t VmmGranularity(int ordinal);
// Physical memory on `ordinal`, mapped at a fresh VA readable/writable by
// every device in `access` (must include `ordinal`).
absl::Status VmmAllocate(int ordinal, size_t bytes, const std::vector<int>& access, VmmBlock* out);
absl::Status VmmExport(const VmmBlock& block, VmmShare* out);
// Imports a peer's heap (pidfd_getfd) and maps it for `ordinal`.
absl::Status VmmImport(const VmmShare& share, int ordinal, VmmBlock* out);
void VmmRelease(VmmBlock* block);

// One NVLink multicast object spanning `devices`, with a VA per device that
// multimem.* instructions address. Single-process helpers; the cross-process
// protocol lives in context.cc (it needs the host exchange callback).
struct McObject {
  CUmemGenericAllocationHandle handle = 0;
  size_t bytes = 0;
  std::vector<int> devices;          // CUDA ordinals, member order
  std::vector<CUdeviceptr> va;       // per entry of `devices` driven here (0 otherwise)
};

bool MulticastSupported(int ordinal);
size_t MulticastGranularity(int num_devices, size_t bytes);

}  // namespace rs

#endif  // REDSYNTH_B200_EXEC_VMM_H_
