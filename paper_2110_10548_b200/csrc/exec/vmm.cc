// CUDA VMM + multicast helpers (see vmm.h).
#include "vmm.h"

#include <cuda_runtime.h>
#include <sys/syscall.h>
#include <unistd.h>

#include <cerrno>
#include <cstring>

#include "absl/strings/str_format.h"

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

namespace rs {

absl::Status CuStatus(CUresult r, const char* what) {
  if (r == CUDA_SUCCESS) return absl::OkStatus();
  const char* s = nullptr;
  drv::cuGetErrorString(r, &s);
  return absl::InternalError(absl::StrFormat("%s: %s (%d)", what, s ? s : "?", static_cast<int>(r)));
}

#define RS_CU(expr)                                   \
  do {                                                \
    absl::Status _s = CuStatus((expr), #expr);        \
    if (!_s.ok()) return _s;                          \
  } while (0)

namespace {

CUmemAllocationProp AllocProp(int ordinal) {
  CUmemAllocationProp p = {};
  p.type = CU_MEM_ALLOCATION_TYPE_PINNED;
  p.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
  p.location.id = ordinal;
  p.requestedHandleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  return p;
}

absl::Status MapFor(VmmBlock* b, const std::vector<int>& access) {
  RS_CU(drv::cuMemAddressReserve(&b->va, b->bytes, 2u << 20, 0, 0));
  RS_CU(drv::cuMemMap(b->va, b->bytes, 0, b->handle, 0));
  std::vector<CUmemAccessDesc> desc(access.size());
  for (size_t i = 0; i < access.size(); ++i) {
    desc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    desc[i].location.id = access[i];
    desc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
  }
  RS_CU(drv::cuMemSetAccess(b->va, b->bytes, desc.data(), desc.size()));
  b->mapped = true;
  return absl::OkStatus();
}

}  // namespace

size_t VmmGranularity(int ordinal) {
  CUmemAllocationProp p = AllocProp(ordinal);
  size_t g = 0;
  if (drv::cuMemGetAllocationGranularity(&g, &p, CU_MEM_ALLOC_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0) {
    g = 2u << 20;
  }
  return g;
}

absl::Status VmmAllocate(int ordinal, size_t bytes, const std::vector<int>& access, VmmBlock* out) {
  RS_CU(drv::cuInit(0));
  CUmemAllocationProp p = AllocProp(ordinal);
  const size_t g = VmmGranularity(ordinal);
  out->bytes = (bytes + g - 1) / g * g;
  RS_CU(drv::cuMemCreate(&out->handle, out->bytes, &p, 0));
  return MapFor(out, access);
}

absl::Status VmmExport(const VmmBlock& block, VmmShare* out) {
  int fd = -1;
  RS_CU(drv::cuMemExportToShareableHandle(&fd, block.handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0));
  out->magic = kVmmMagic;
  out->pid = static_cast<int32_t>(getpid());
  out->fd = fd;
  out->pad = 0;
  out->bytes = block.bytes;
  return absl::OkStatus();
}

absl::Status VmmImport(const VmmShare& share, int ordinal, VmmBlock* out) {
  if (share.magic != kVmmMagic) return absl::InvalidArgumentError("peer handle is not a VMM heap share");
  const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, share.pid, 0));
  if (pidfd < 0) {
    return absl::UnavailableError(absl::StrFormat("pidfd_open(%d): %s", share.pid, std::strerror(errno)));
  }
  const int fd = static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, share.fd, 0));
  const int err = errno;
  close(pidfd);
  if (fd < 0) {
    return absl::UnavailableError(
        absl::StrFormat("pidfd_getfd(pid %d, fd %d): %s", share.pid, share.fd, std::strerror(err)));
  }
  out->bytes = share.bytes;
  const CUresult r = drv::cuMemImportFromShareableHandle(
      &out->handle, reinterpret_cast<void*>(static_cast<intptr_t>(fd)), CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR);
  close(fd);
  RS_CU(r);
  return MapFor(out, {ordinal});
}

void VmmRelease(VmmBlock* b) {
  if (b->mapped) {
    drv::cuMemUnmap(b->va, b->bytes);
    drv::cuMemAddressFree(b->va, b->bytes);
    b->mapped = false;
  }
  if (b->handle) {
    drv::cuMemRelease(b->handle);
    b->handle = 0;
  }
}

bool MulticastSupported(int ordinal) {
  if (drv::cuInit(0) != CUDA_SUCCESS) return false;
  CUdevice dev;
  if (drv::cuDeviceGet(&dev, ordinal) != CUDA_SUCCESS) return false;
  int v = 0;
  if (drv::cuDeviceGetAttribute(&v, CU_DEVICE_ATTRIBUTE_MULTICAST_SUPPORTED, dev) != CUDA_SUCCESS) return false;
  return v != 0;
}

size_t MulticastGranularity(int num_devices, size_t bytes) {
  CUmulticastObjectProp prop = {};
  prop.numDevices = static_cast<unsigned>(num_devices);
  prop.size = bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  size_t g = 0;
  if (drv::cuMulticastGetGranularity(&g, &prop, CU_MULTICAST_GRANULARITY_MINIMUM) != CUDA_SUCCESS || g == 0) {
    g = 2u << 20;
  }
  return g;
}

}  // namespace rs

namespace rs::drv {

void* Resolve(const char* name) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult status{};
  if (cudaGetDriverEntryPoint(name, &fn, cudaEnableDefault, &status) != cudaSuccess ||
      status != cudaDriverEntryPointSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return fn;
}

}  // namespace rs::drv
