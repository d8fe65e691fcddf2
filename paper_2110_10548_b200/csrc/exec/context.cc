// Executor contexts: per-rank heaps (slot buffers + barrier flags), peer
// mappings (CUDA peer access in one process, CUDA IPC across processes) and
// streams.
#include <sys/syscall.h>
#include <unistd.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>

#ifndef SYS_pidfd_open
#define SYS_pidfd_open 434
#endif
#ifndef SYS_pidfd_getfd
#define SYS_pidfd_getfd 438
#endif

#include "absl/strings/str_format.h"
#include "exec_internal.h"

namespace rs {

absl::Status CudaStatus(cudaError_t err, const char* what) {
  if (err == cudaSuccess) return absl::OkStatus();
  if (err == cudaErrorNoDevice || err == cudaErrorInsufficientDriver) {
    return absl::UnavailableError(absl::StrFormat("%s: %s", what, cudaGetErrorString(err)));
  }
  return absl::InternalError(absl::StrFormat("%s: %s", what, cudaGetErrorString(err)));
}

#define RS_CUDA(expr)                                          \
  do {                                                         \
    absl::Status _s = CudaStatus((expr), #expr);               \
    if (!_s.ok()) return _s;                                   \
  } while (0)

std::vector<int> Context::DrivenRanks() const {
  std::vector<int> out;
  for (int r = 0; r < world; ++r)
    if (ranks[r].driven) out.push_back(r);
  return out;
}

namespace {

size_t RoundUp(size_t x, size_t a) { return (x + a - 1) / a * a; }

absl::Status AllocateRank(Context* ctx, int r) {
  Rank& rank = ctx->ranks[r];
  RS_CUDA(cudaSetDevice(rank.ordinal));
  rank.heap_bytes = ctx->flag_offset[r] + ctx->flag_bytes[r];  // slots, LL area, flags (AssignPositions)
  if (ctx->use_vmm) {
    // cuMemCreate'd heap: shareable as a POSIX fd and bindable to multicast.
    std::vector<int> access{rank.ordinal};
    if (ctx->self_rank < 0) {
      for (const Rank& other : ctx->ranks)
        if (other.ordinal != rank.ordinal) access.push_back(other.ordinal);
    }
    absl::Status s = VmmAllocate(rank.ordinal, rank.heap_bytes, access, &rank.vmm);
    if (!s.ok()) return s;
    rank.heap_bytes = rank.vmm.bytes;
    rank.heap = reinterpret_cast<char*>(rank.vmm.va);
  } else {
    void* heap = nullptr;
    RS_CUDA(cudaMalloc(&heap, rank.heap_bytes));
    rank.heap = static_cast<char*>(heap);
  }
  RS_CUDA(cudaMemset(rank.heap, 0, kDataOffset));
  if (ctx->ll_capacity > 0 || ctx->flag_bytes[r] > 0) {
    RS_CUDA(cudaMemset(rank.heap + ctx->ll_offset[r], 0, rank.heap_bytes - ctx->ll_offset[r]));
  }
  const uint64_t first_epoch = 1;
  RS_CUDA(cudaMemcpy(rank.heap + kEpochOffset, &first_epoch, sizeof(first_epoch), cudaMemcpyHostToDevice));
  RS_CUDA(cudaStreamCreateWithFlags(&rank.stream, cudaStreamNonBlocking));
  RS_CUDA(cudaDeviceGetAttribute(&rank.sm_count, cudaDevAttrMultiProcessorCount, rank.ordinal));
  rank.driven = true;
  rank.view.assign(ctx->world, nullptr);
  rank.view[r] = rank.heap;
  return absl::OkStatus();
}

absl::Status CheckCommon(int K, size_t max_bytes) {
  if (K < 1 || K > 4096) return absl::InvalidArgumentError("K must be in [1, 4096]");
  if (max_bytes == 0) return absl::InvalidArgumentError("max_bytes must be positive");
  return absl::OkStatus();
}

// Slot positions within their rank's heap, and the scratch budget: the push
// variant lands one copy per group member in the owner's scratch, so
// cross-GPU contexts reserve min(K, 8) regions per slot (RS_SCRATCH_REGIONS
// overrides; 0 disables the push variant).
void AssignPositions(Context* ctx) {
  std::vector<int> next(ctx->world, 0);
  ctx->slot_position.assign(ctx->K, 0);
  for (int d = 0; d < ctx->K; ++d) ctx->slot_position[d] = next[ctx->slot_rank[d]]++;
  ctx->scratch_regions = ctx->is_virtual ? ctx->K : (ctx->world > 1 ? std::min(ctx->K, 8) : 0);
  if (const char* env = std::getenv("RS_SCRATCH_REGIONS")) {
    const int v = std::atoi(env);
    if (v >= 0) ctx->scratch_regions = v;
  }
  // One-shot (LL) area after the slots: RS_LL_CAPACITY payload bytes per
  // (sender, parity) region (0 disables); RS_LL_MAX_BYTES the step budget.
  if (ctx->world > 1) {
    ctx->ll_capacity = 512u << 10;
    ctx->ll_max_bytes = 256u << 10;
    if (const char* env = std::getenv("RS_LL_CAPACITY")) ctx->ll_capacity = std::strtoull(env, nullptr, 10) & ~7ull;
    if (const char* env = std::getenv("RS_LL_MAX_BYTES")) ctx->ll_max_bytes = std::strtoull(env, nullptr, 10);
    if (const char* env = std::getenv("RS_LL_TOTAL_BYTES")) ctx->ll_total_bytes = std::strtoull(env, nullptr, 10);
  }
  if (const char* env = std::getenv("RS_RECV_PIECE")) ctx->recv_piece_bytes = std::strtoull(env, nullptr, 10);
  if (const char* env = std::getenv("RS_FLAG_CHUNK")) {
    const uint64_t c = std::strtoull(env, nullptr, 10) & ~15ull;
    if (c >= (16u << 10)) ctx->flag_chunk = c;
  }
  ctx->ll_offset.assign(ctx->world, 0);
  ctx->flag_offset.assign(ctx->world, 0);
  ctx->flag_bytes.assign(ctx->world, 0);
  for (int r = 0; r < ctx->world; ++r) {
    ctx->ll_offset[r] = kDataOffset + static_cast<size_t>(next[r]) * (1 + ctx->scratch_regions) * ctx->slot_stride;
    ctx->flag_offset[r] = ctx->ll_offset[r] + static_cast<size_t>(ctx->world) * 2 * ctx->LLRegionBytes();
    if (ctx->world > 1) {
      // per (slot, region): its chunks, doubled plus slack for parts split
      // into several row ranges (each rounds up to whole chunks)
      const uint64_t chunks = 2 * ((ctx->slot_stride + ctx->flag_chunk - 1) / ctx->flag_chunk) + 64;
      ctx->flag_bytes[r] = static_cast<uint64_t>(next[r]) * (1 + ctx->scratch_regions) * chunks * sizeof(uint64_t);
    }
  }
}

// NVLS needs a VMM heap; opt in with RS_NVLS=1 (multi-GPU contexts whose
// GPUs support multicast). Every rank of a job must make the same choice.
void DecideNvls(Context* ctx, const std::vector<int>& ordinals) {
  const char* env = std::getenv("RS_NVLS");
  if (!env || std::atoi(env) == 0 || ctx->world < 2) return;
  for (int o : ordinals)
    if (!MulticastSupported(o)) return;
  ctx->use_vmm = true;
  ctx->nvls = true;
  if (const char* g = std::getenv("RS_NVLS_MIN_GROUP")) ctx->nvls_min_group = std::max(2, std::atoi(g));
  if (const char* b = std::getenv("RS_NVLS_MIN_BYTES")) {
    ctx->nvls_min_bytes = std::strtoull(b, nullptr, 10);
    ctx->nvls_min_bytes_n8 = ctx->nvls_min_bytes;
  }
}

void ReadTimeoutEnv(Context* ctx) {
  if (const char* env = std::getenv("RS_BARRIER_TIMEOUT_S")) {
    const double s = std::atof(env);
    if (s > 0) ctx->timeout_ns = static_cast<uint64_t>(s * 1e9);
  }
  if (const char* env = std::getenv("RS_PUSH_MIN_BYTES")) {
    ctx->push_min_bytes = std::strtoull(env, nullptr, 10);
  }
  if (const char* env = std::getenv("RS_PUSH_MAX_GPUS")) ctx->push_max_gpus = std::atoi(env);
  if (const char* env = std::getenv("RS_PUSH_WAVE_BYTES")) {
    ctx->push_wave_bytes = std::strtoull(env, nullptr, 10) & ~15ull;
  }
  if (const char* env = std::getenv("RS_WAVE_LAG")) ctx->wave_lag = std::max(0, std::atoi(env));
  if (const char* env = std::getenv("RS_REDUCE_MODE")) {
    const int m = std::atoi(env);
    if (m >= kReduceAuto && m <= kReducePushRootPulled) ctx->reduce_mode = m;
  }
}

}  // namespace

absl::Status CreateContext(int K, const int* ordinals, size_t max_bytes, Context** out) {
  absl::Status ok = CheckCommon(K, max_bytes);
  if (!ok.ok()) return ok;
  if (ordinals == nullptr) return absl::InvalidArgumentError("cuda_ordinals is null");
  int devices = 0;
  RS_CUDA(cudaGetDeviceCount(&devices));
  auto ctx = std::make_unique<Context>();
  ctx->K = K;
  ctx->max_bytes = max_bytes;
  ctx->slot_stride = RoundUp(max_bytes, kSlotAlign);
  ReadTimeoutEnv(ctx.get());
  // Ranks = distinct ordinals in order of first appearance.
  std::vector<int> rank_ordinal;
  ctx->slot_rank.resize(K);
  for (int d = 0; d < K; ++d) {
    if (ordinals[d] < 0 || ordinals[d] >= devices) {
      return absl::InvalidArgumentError(
          absl::StrFormat("slot %d: CUDA ordinal %d out of range (%d devices)", d, ordinals[d], devices));
    }
    auto it = std::find(rank_ordinal.begin(), rank_ordinal.end(), ordinals[d]);
    if (it == rank_ordinal.end()) {
      rank_ordinal.push_back(ordinals[d]);
      it = rank_ordinal.end() - 1;
    }
    ctx->slot_rank[d] = static_cast<int>(it - rank_ordinal.begin());
  }
  ctx->world = static_cast<int>(rank_ordinal.size());
  if (ctx->world > RS_MAX_RANKS) {
    return absl::InvalidArgumentError(absl::StrFormat("at most %d GPUs per context", RS_MAX_RANKS));
  }
  AssignPositions(ctx.get());
  ctx->ranks.resize(ctx->world);
  for (int r = 0; r < ctx->world; ++r) ctx->ranks[r].ordinal = rank_ordinal[r];
  DecideNvls(ctx.get(), rank_ordinal);
  for (int r = 0; r < ctx->world; ++r) {
    absl::Status s = AllocateRank(ctx.get(), r);
    if (!s.ok()) {
      DestroyContext(ctx.release());
      return s;
    }
  }
  // One process: peers are addressed directly (UVA) once peer access is on.
  for (int r = 0; r < ctx->world; ++r) {
    RS_CUDA(cudaSetDevice(ctx->ranks[r].ordinal));
    for (int q = 0; q < ctx->world; ++q) {
      if (q == r) continue;
      int can = 0;
      RS_CUDA(cudaDeviceCanAccessPeer(&can, ctx->ranks[r].ordinal, ctx->ranks[q].ordinal));
      if (!can) {
        return absl::UnavailableError(absl::StrFormat("GPU %d cannot access GPU %d",
                                                      ctx->ranks[r].ordinal, ctx->ranks[q].ordinal));
      }
      cudaError_t e = cudaDeviceEnablePeerAccess(ctx->ranks[q].ordinal, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else {
        RS_CUDA(e);
      }
      ctx->ranks[r].view[q] = ctx->ranks[q].heap;
    }
  }
  ctx->peers_open = true;
  *out = ctx.release();
  return absl::OkStatus();
}

absl::Status CreateRankContext(int K, const int* slot_rank, int world, int rank, int ordinal,
                               size_t max_bytes, Context** out) {
  absl::Status ok = CheckCommon(K, max_bytes);
  if (!ok.ok()) return ok;
  if (world < 1 || world > RS_MAX_RANKS) {
    return absl::InvalidArgumentError(absl::StrFormat("world_size must be in [1, %d]", RS_MAX_RANKS));
  }
  if (rank < 0 || rank >= world) return absl::InvalidArgumentError("rank out of range");
  if (slot_rank == nullptr) return absl::InvalidArgumentError("slot_rank is null");
  auto ctx = std::make_unique<Context>();
  ctx->K = K;
  ctx->max_bytes = max_bytes;
  ctx->slot_stride = RoundUp(max_bytes, kSlotAlign);
  ctx->world = world;
  ctx->self_rank = rank;
  ReadTimeoutEnv(ctx.get());
  ctx->slot_rank.assign(slot_rank, slot_rank + K);
  for (int d = 0; d < K; ++d) {
    if (slot_rank[d] < 0 || slot_rank[d] >= world) {
      return absl::InvalidArgumentError(absl::StrFormat("slot %d: rank %d out of range", d, slot_rank[d]));
    }
  }
  AssignPositions(ctx.get());
  ctx->ranks.resize(world);
  ctx->ranks[rank].ordinal = ordinal;
  DecideNvls(ctx.get(), {ordinal});
  absl::Status s = AllocateRank(ctx.get(), rank);
  if (!s.ok()) {
    DestroyContext(ctx.release());
    return s;
  }
  ctx->peers_open = world == 1;
  *out = ctx.release();
  return absl::OkStatus();
}

absl::Status CreateEmulatedContext(int K, const int* slot_rank, int world, int ordinal, size_t max_bytes,
                                   Context** out) {
  absl::Status ok = CheckCommon(K, max_bytes);
  if (!ok.ok()) return ok;
  if (world < 2 || world > RS_MAX_RANKS) {
    return absl::InvalidArgumentError(absl::StrFormat("world_size must be in [2, %d]", RS_MAX_RANKS));
  }
  if (slot_rank == nullptr) return absl::InvalidArgumentError("slot_rank is null");
  int devices = 0;
  RS_CUDA(cudaGetDeviceCount(&devices));
  if (ordinal < 0 || ordinal >= devices) return absl::InvalidArgumentError("cuda_ordinal out of range");
  auto ctx = std::make_unique<Context>();
  ctx->K = K;
  ctx->max_bytes = max_bytes;
  ctx->slot_stride = RoundUp(max_bytes, kSlotAlign);
  ctx->world = world;
  ctx->emulated = true;
  ReadTimeoutEnv(ctx.get());
  ctx->slot_rank.assign(slot_rank, slot_rank + K);
  for (int d = 0; d < K; ++d) {
    if (slot_rank[d] < 0 || slot_rank[d] >= world) {
      return absl::InvalidArgumentError(absl::StrFormat("slot %d: rank %d out of range", d, slot_rank[d]));
    }
  }
  AssignPositions(ctx.get());
  ctx->ranks.resize(world);
  for (int r = 0; r < world; ++r) ctx->ranks[r].ordinal = ordinal;
  for (int r = 0; r < world; ++r) {
    absl::Status s = AllocateRank(ctx.get(), r);
    if (!s.ok()) {
      DestroyContext(ctx.release());
      return s;
    }
  }
  for (int r = 0; r < world; ++r)
    for (int q = 0; q < world; ++q) ctx->ranks[r].view[q] = ctx->ranks[q].heap;
  ctx->peers_open = true;
  *out = ctx.release();
  return absl::OkStatus();
}

absl::Status CreateVirtualContext(int K, const int* slot_rank, int world, Context** out) {
  if (K < 1 || K > 4096) return absl::InvalidArgumentError("K must be in [1, 4096]");
  if (world < 1 || world > RS_MAX_RANKS) {
    return absl::InvalidArgumentError(absl::StrFormat("world_size must be in [1, %d]", RS_MAX_RANKS));
  }
  auto ctx = std::make_unique<Context>();
  ctx->K = K;
  ctx->max_bytes = ~size_t{0} >> 1;
  ctx->world = world;
  ctx->is_virtual = true;
  ctx->peers_open = true;
  ctx->slot_rank.assign(slot_rank, slot_rank + K);
  for (int d = 0; d < K; ++d) {
    if (slot_rank[d] < 0 || slot_rank[d] >= world) {
      return absl::InvalidArgumentError(absl::StrFormat("slot %d: rank %d out of range", d, slot_rank[d]));
    }
  }
  AssignPositions(ctx.get());
  ReadTimeoutEnv(ctx.get());
  ctx->ranks.resize(world);
  *out = ctx.release();
  return absl::OkStatus();
}

absl::Status IpcHandle(Context* ctx, void* out) {
  if (ctx->self_rank < 0) return absl::InvalidArgumentError("not a per-rank context");
  Rank& me = ctx->ranks[ctx->self_rank];
  RS_CUDA(cudaSetDevice(me.ordinal));
  std::memset(out, 0, RS_IPC_HANDLE_BYTES);
  if (ctx->use_vmm) {
    VmmShare share{};
    absl::Status s = VmmExport(me.vmm, &share);
    if (!s.ok()) return s;
    static_assert(sizeof(share) <= RS_IPC_HANDLE_BYTES, "share size");
    std::memcpy(out, &share, sizeof(share));
    return absl::OkStatus();
  }
  cudaIpcMemHandle_t h;
  RS_CUDA(cudaIpcGetMemHandle(&h, me.heap));
  static_assert(sizeof(h) == RS_IPC_HANDLE_BYTES, "IPC handle size");
  std::memcpy(out, &h, sizeof(h));
  return absl::OkStatus();
}

absl::Status OpenPeers(Context* ctx, const void* handles) {
  if (ctx->self_rank < 0) return absl::InvalidArgumentError("not a per-rank context");
  if (ctx->peers_open) return absl::OkStatus();
  Rank& me = ctx->ranks[ctx->self_rank];
  RS_CUDA(cudaSetDevice(me.ordinal));
  const char* bytes = static_cast<const char*>(handles);
  for (int q = 0; q < ctx->world; ++q) {
    if (q == ctx->self_rank) continue;
    const char* blob = bytes + static_cast<size_t>(q) * RS_IPC_HANDLE_BYTES;
    if (ctx->use_vmm) {
      VmmShare share;
      std::memcpy(&share, blob, sizeof(share));
      VmmBlock block;
      absl::Status s = VmmImport(share, me.ordinal, &block);
      if (!s.ok()) return s;
      me.imported.push_back(block);
      me.view[q] = reinterpret_cast<char*>(block.va);
      continue;
    }
    cudaIpcMemHandle_t h;
    std::memcpy(&h, blob, sizeof(h));
    void* p = nullptr;
    RS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    me.view[q] = static_cast<char*>(p);
  }
  ctx->peers_open = true;
  return absl::OkStatus();
}

absl::Status Synchronize(Context* ctx) {
  // Plans usually run on caller streams (rs_plan_run streams, torch's current
  // stream), so wait for the whole device, not just the context's streams.
  // The timeout flag is reported once and then cleared, so later healthy
  // runs synchronize cleanly.
  absl::Status first = absl::OkStatus();
  for (int r : ctx->DrivenRanks()) {
    Rank& rank = ctx->ranks[r];
    RS_CUDA(cudaSetDevice(rank.ordinal));
    RS_CUDA(cudaDeviceSynchronize());
    int err = 0;
    RS_CUDA(cudaMemcpy(&err, rank.heap + kErrorOffset, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      RS_CUDA(cudaMemset(rank.heap + kErrorOffset, 0, sizeof(int)));
      if (first.ok()) {
        first = err == 1 ? absl::InternalError(absl::StrFormat(
                               "rank %d: inter-GPU barrier timed out (a peer never reached the step); results are "
                               "invalid", r))
                         : absl::InternalError(absl::StrFormat(
                               "rank %d: checked-build assertion %d failed in the step kernel (see the device "
                               "printf); results are invalid", r, err));
      }
    }
  }
  return first;
}

absl::Status DestroyContext(Context* ctx) {
  if (ctx == nullptr) return absl::OkStatus();
  for (int r = 0; r < ctx->world; ++r) {
    Rank& rank = ctx->ranks[r];
    if (!rank.driven) continue;
    cudaSetDevice(rank.ordinal);
    if (rank.stream) cudaStreamSynchronize(rank.stream);
    if (ctx->self_rank >= 0 && !ctx->use_vmm) {
      for (int q = 0; q < ctx->world; ++q)
        if (q != r && rank.view.size() > static_cast<size_t>(q) && rank.view[q]) cudaIpcCloseMemHandle(rank.view[q]);
    }
    if (rank.stream) cudaStreamDestroy(rank.stream);
  }
  // Multicast objects first (they hold bindings to the heaps).
  for (auto& [slots, mc] : ctx->mc_groups) {
    for (int r = 0; r < ctx->world; ++r) {
      if (!ctx->ranks[r].driven || !mc->va[r]) continue;
      cudaSetDevice(ctx->ranks[r].ordinal);
      cudaDeviceSynchronize();
      drv::cuMemUnmap(mc->va[r], mc->bytes);
      drv::cuMemAddressFree(mc->va[r], mc->bytes);
      if (ctx->self_rank < 0) break;  // one mapping shared by every device
    }
    for (int d : slots) {
      const int r = ctx->slot_rank[d];
      if (!ctx->ranks[r].driven) continue;
      CUdevice dev;
      if (drv::cuDeviceGet(&dev, ctx->ranks[r].ordinal) == CUDA_SUCCESS) {
        drv::cuMulticastUnbind(mc->handle, dev, 0, mc->bytes);
      }
    }
    if (mc->handle) drv::cuMemRelease(mc->handle);
  }
  for (int r = 0; r < ctx->world; ++r) {
    Rank& rank = ctx->ranks[r];
    if (!rank.driven) continue;
    cudaSetDevice(rank.ordinal);
    for (VmmBlock& b : rank.imported) VmmRelease(&b);
    if (ctx->use_vmm) {
      VmmRelease(&rank.vmm);
    } else if (rank.heap) {
      cudaFree(rank.heap);
    }
  }
  delete ctx;
  return absl::OkStatus();
}

namespace {

// Collective host exchange (all ranks, same order): send `bytes` bytes,
// receive world * bytes. Required for multi-process multicast setup.
absl::Status Exchange(Context* ctx, const void* send, size_t bytes, std::vector<char>* recv) {
  recv->assign(bytes * ctx->world, 0);
  if (ctx->exchange == nullptr) {
    return absl::FailedPreconditionError(
        "multi-process NVLS setup needs the host exchange callback (rs_ctx_set_exchange)");
  }
  if (ctx->exchange(send, bytes, recv->data(), ctx->exchange_user) != 0) {
    return absl::InternalError("host exchange callback failed");
  }
  return absl::OkStatus();
}

// NVLS self-check (every new multicast object, before any plan uses it):
// each member's first kSelfCheckBytes are saved, filled with small integers
// (exact f32 sums), all-reduced through the switch by the members (each its
// slice, the instructions the NVLS tasks use), compared with the expected
// sums and restored. Any failure — a launch error, a wrong sum, a rank that
// cannot run it — makes every rank drop the object and fall back to P2P.
constexpr size_t kSelfCheckBytes = 64u << 10;

float SelfCheckValue(int slot, size_t e) { return static_cast<float>(slot % 5 + 1) + static_cast<float>(e % 7); }

absl::Status NvlsSelfCheck(Context* ctx, McGroup* mc, const std::vector<int>& slots,
                           absl::Status (*barrier)(Context*, int32_t ok, bool* all_ok)) {
  const size_t elems = kSelfCheckBytes / sizeof(float);
  const int n = static_cast<int>(slots.size());
  std::vector<int> mine;  // indices into slots of the members driven here
  for (int i = 0; i < n; ++i)
    if (ctx->ranks[ctx->slot_rank[slots[i]]].driven) mine.push_back(i);
  std::vector<void*> saved(mine.size(), nullptr);
  int32_t ok = 1;
  std::vector<float> host(elems);
  bool all_ok = false;
  // 0. quiesce: runs enqueued earlier (on any stream, by any rank) may still
  //    touch the slot buffers
  for (const Rank& rank : ctx->ranks) {
    if (!rank.driven) continue;
    ok &= cudaSetDevice(rank.ordinal) == cudaSuccess && cudaDeviceSynchronize() == cudaSuccess;
  }
  absl::Status bs = barrier(ctx, ok, &all_ok);
  if (!bs.ok()) return bs;
  // 1. save + fill
  for (size_t k = 0; k < mine.size() && ok; ++k) {
    const int d = slots[mine[k]];
    const int r = ctx->slot_rank[d];
    ok &= cudaSetDevice(ctx->ranks[r].ordinal) == cudaSuccess;
    ok &= ok && cudaMalloc(&saved[k], kSelfCheckBytes) == cudaSuccess;
    ok &= ok && cudaMemcpy(saved[k], ctx->SlotPtr(r, d), kSelfCheckBytes, cudaMemcpyDeviceToDevice) == cudaSuccess;
    for (size_t e = 0; e < elems; ++e) host[e] = SelfCheckValue(d, e);
    ok &= ok && cudaMemcpy(ctx->SlotPtr(r, d), host.data(), kSelfCheckBytes, cudaMemcpyHostToDevice) == cudaSuccess;
    ok &= ok && cudaDeviceSynchronize() == cudaSuccess;
  }
  bs = barrier(ctx, ok, &all_ok);
  if (!bs.ok()) return bs;
  // 2. reduce through the switch: member i handles slice i
  if (all_ok) {
    for (size_t k = 0; k < mine.size() && ok; ++k) {
      const int i = mine[k];
      const int r = ctx->slot_rank[slots[i]];
      const uint64_t lo = (kSelfCheckBytes * i / n) & ~uint64_t{15};
      const uint64_t hi = i + 1 == n ? kSelfCheckBytes : (kSelfCheckBytes * (i + 1) / n) & ~uint64_t{15};
      ok &= cudaSetDevice(ctx->ranks[r].ordinal) == cudaSuccess;
      ok &= ok && LaunchNvlsSelfCheck(reinterpret_cast<char*>(mc->va[r]), lo, hi, nullptr) == cudaSuccess;
    }
    for (size_t k = 0; k < mine.size(); ++k) {
      cudaSetDevice(ctx->ranks[ctx->slot_rank[slots[mine[k]]]].ordinal);
      ok &= cudaDeviceSynchronize() == cudaSuccess;
    }
    bs = barrier(ctx, ok, &all_ok);
    if (!bs.ok()) return bs;
  }
  // 3. compare
  if (all_ok) {
    for (size_t k = 0; k < mine.size() && ok; ++k) {
      const int d = slots[mine[k]];
      const int r = ctx->slot_rank[d];
      cudaSetDevice(ctx->ranks[r].ordinal);
      ok &= cudaMemcpy(host.data(), ctx->SlotPtr(r, d), kSelfCheckBytes, cudaMemcpyDeviceToHost) == cudaSuccess;
      for (size_t e = 0; e < elems && ok; ++e) {
        float want = 0;
        for (int m : slots) want += SelfCheckValue(m, e);
        ok &= host[e] == want;
      }
    }
    bs = barrier(ctx, ok, &all_ok);
    if (!bs.ok()) return bs;
  }
  // 4. restore
  for (size_t k = 0; k < mine.size(); ++k) {
    if (!saved[k]) continue;
    const int d = slots[mine[k]];
    const int r = ctx->slot_rank[d];
    cudaSetDevice(ctx->ranks[r].ordinal);
    cudaMemcpy(ctx->SlotPtr(r, d), saved[k], kSelfCheckBytes, cudaMemcpyDeviceToDevice);
    cudaFree(saved[k]);
  }
  cudaGetLastError();
  if (!all_ok) return absl::InternalError("NVLS self-check failed (multicast sums wrong or not runnable)");
  return absl::OkStatus();
}

// Barriers of the self-check: one process sees every member's verdict
// directly; one process per GPU all-gathers the verdicts (all ranks take
// part, members or not, like the other setup exchanges).
absl::Status LocalBarrier(Context*, int32_t ok, bool* all_ok) {
  *all_ok = ok != 0;
  return absl::OkStatus();
}

absl::Status ExchangeBarrier(Context* ctx, int32_t ok, bool* all_ok) {
  std::vector<char> all;
  absl::Status s = Exchange(ctx, &ok, sizeof(ok), &all);
  if (!s.ok()) return s;
  *all_ok = true;
  for (int r = 0; r < ctx->world; ++r) {
    int32_t v;
    std::memcpy(&v, all.data() + r * sizeof(int32_t), sizeof(v));
    *all_ok = *all_ok && v != 0;
  }
  return absl::OkStatus();
}

struct McShare {
  int32_t pid;
  int32_t fd;
  int32_t ok;
  int32_t pad;
};

}  // namespace

absl::Status EnsureMulticast(Context* ctx, const std::vector<int>& slots, int* index) {
  auto found = ctx->mc_groups.find(slots);
  if (found != ctx->mc_groups.end()) {
    for (size_t i = 0; i < ctx->mc_index.size(); ++i)
      if (ctx->mc_index[i] == found->second.get()) *index = static_cast<int>(i);
    return absl::OkStatus();
  }
  auto mc = std::make_unique<McGroup>();
  mc->slots = slots;
  mc->va.assign(ctx->world, 0);
  if (ctx->is_virtual) {  // planning only: record the group, no CUDA objects
    *index = static_cast<int>(ctx->mc_index.size());
    ctx->mc_index.push_back(mc.get());
    ctx->mc_groups[slots] = std::move(mc);
    return absl::OkStatus();
  }
  // Everything created below is released on every early return (a failed
  // NVLS setup falls back to P2P and must not leak switch resources).
  struct Cleanup {
    McGroup* mc;
    std::vector<std::pair<int, CUdevice>> bound;  // (ordinal, device) bound to mc
    std::vector<std::pair<int, CUdeviceptr>> mapped;  // (ordinal, va)
    int fd = -1;
    bool armed = true;
    ~Cleanup() {
      if (fd >= 0) close(fd);
      if (!armed) return;
      for (auto [ord, va] : mapped) {
        cudaSetDevice(ord);
        drv::cuMemUnmap(va, mc->bytes);
        drv::cuMemAddressFree(va, mc->bytes);
      }
      for (auto [ord, dev] : bound) {
        cudaSetDevice(ord);
        drv::cuMulticastUnbind(mc->handle, dev, 0, mc->bytes);
      }
      if (mc->handle) drv::cuMemRelease(mc->handle);
      std::fill(mc->va.begin(), mc->va.end(), 0);
    }
  } guard{mc.get()};
  const int n = static_cast<int>(slots.size());
  const size_t gran = MulticastGranularity(n, ctx->max_bytes);
  mc->bytes = (ctx->max_bytes + gran - 1) / gran * gran;
  if (mc->bytes > ctx->slot_stride) return absl::InternalError("multicast size exceeds slot stride");
  CUmulticastObjectProp prop = {};
  prop.numDevices = static_cast<unsigned>(n);
  prop.size = mc->bytes;
  prop.handleTypes = CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR;
  auto device_of = [&](int r) {
    CUdevice dev = 0;
    drv::cuDeviceGet(&dev, ctx->ranks[r].ordinal);
    return dev;
  };
  auto bind = [&](int r, int slot) -> absl::Status {
    RS_CUDA(cudaSetDevice(ctx->ranks[r].ordinal));
    absl::Status s = CuStatus(
        drv::cuMulticastBindMem(mc->handle, 0, ctx->ranks[r].vmm.handle, ctx->SlotOffset(slot, -1), mc->bytes, 0),
        "cuMulticastBindMem");
    if (s.ok()) guard.bound.push_back({ctx->ranks[r].ordinal, device_of(r)});
    return s;
  };
  auto map_va = [&](const std::vector<int>& access, CUdeviceptr* va) -> absl::Status {
    absl::Status s = CuStatus(drv::cuMemAddressReserve(va, mc->bytes, gran, 0, 0), "reserve multicast VA");
    if (!s.ok()) return s;
    s = CuStatus(drv::cuMemMap(*va, mc->bytes, 0, mc->handle, 0), "map multicast VA");
    if (!s.ok()) {
      drv::cuMemAddressFree(*va, mc->bytes);
      *va = 0;
      return s;
    }
    int ord = 0;
    cudaGetDevice(&ord);
    guard.mapped.push_back({ord, *va});
    std::vector<CUmemAccessDesc> desc(access.size());
    for (size_t i = 0; i < access.size(); ++i) {
      desc[i].location.type = CU_MEM_LOCATION_TYPE_DEVICE;
      desc[i].location.id = access[i];
      desc[i].flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    }
    return CuStatus(drv::cuMemSetAccess(*va, mc->bytes, desc.data(), desc.size()), "multicast access");
  };

  if (ctx->self_rank < 0) {
    // One process: create, add every member GPU, bind each member's slot
    // buffer, map one VA usable by all members.
    absl::Status s = CuStatus(drv::cuMulticastCreate(&mc->handle, &prop), "cuMulticastCreate");
    if (!s.ok()) return s;
    std::vector<int> access;
    for (int d : slots) {
      const int r = ctx->slot_rank[d];
      s = CuStatus(drv::cuMulticastAddDevice(mc->handle, device_of(r)), "cuMulticastAddDevice");
      if (!s.ok()) return s;
      access.push_back(ctx->ranks[r].ordinal);
    }
    for (int d : slots) {
      s = bind(ctx->slot_rank[d], d);
      if (!s.ok()) return s;
    }
    CUdeviceptr va = 0;
    s = map_va(access, &va);
    if (!s.ok()) return s;
    for (int d : slots) mc->va[ctx->slot_rank[d]] = va;
  } else {
    // One process per GPU: the first member's rank creates and shares the
    // object (fd via pidfd_getfd); every member adds its GPU, then binds its
    // slot and maps its own VA. All ranks take part in the exchanges.
    const int me = ctx->self_rank;
    const int creator = ctx->slot_rank[slots[0]];
    bool member = false;
    int my_slot = -1;
    for (int d : slots) {
      if (ctx->slot_rank[d] == me) {
        member = true;
        my_slot = d;
      }
    }
    McShare mine{};
    absl::Status s;
    if (me == creator) {
      s = CuStatus(drv::cuMulticastCreate(&mc->handle, &prop), "cuMulticastCreate");
      if (s.ok()) {
        int fd = -1;
        s = CuStatus(drv::cuMemExportToShareableHandle(&fd, mc->handle, CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR, 0),
                     "export multicast");
        mine = McShare{static_cast<int32_t>(getpid()), fd, s.ok() ? 1 : 0, 0};
        guard.fd = fd;
      }
    }
    std::vector<char> all;
    absl::Status xs = Exchange(ctx, &mine, sizeof(mine), &all);
    if (!xs.ok()) return xs;
    if (!s.ok()) return s;
    McShare theirs;
    std::memcpy(&theirs, all.data() + static_cast<size_t>(creator) * sizeof(McShare), sizeof(theirs));
    if (!theirs.ok) return absl::InternalError("multicast creation failed on the creator rank");
    int32_t added = 1;
    if (member && me != creator) {
      VmmShare vs{kVmmMagic, theirs.pid, theirs.fd, 0, mc->bytes};
      // Reuse the fd import path (pidfd_getfd) without mapping.
      const int pidfd = static_cast<int>(syscall(SYS_pidfd_open, vs.pid, 0));
      const int fd = pidfd < 0 ? -1 : static_cast<int>(syscall(SYS_pidfd_getfd, pidfd, vs.fd, 0));
      if (pidfd >= 0) close(pidfd);
      if (fd < 0) {
        added = 0;
        s = absl::UnavailableError("pidfd_getfd failed for the multicast handle");
      } else {
        s = CuStatus(drv::cuMemImportFromShareableHandle(&mc->handle, reinterpret_cast<void*>(static_cast<intptr_t>(fd)),
                                                    CU_MEM_HANDLE_TYPE_POSIX_FILE_DESCRIPTOR),
                     "import multicast");
        close(fd);
      }
    }
    if (member && s.ok()) {
      s = CuStatus(drv::cuMulticastAddDevice(mc->handle, device_of(me)), "cuMulticastAddDevice");
      added = s.ok() ? 1 : 0;
    }
    xs = Exchange(ctx, &added, sizeof(added), &all);
    if (!xs.ok()) return xs;
    for (int r = 0; r < ctx->world; ++r) {
      int32_t v;
      std::memcpy(&v, all.data() + r * sizeof(int32_t), sizeof(v));
      if (!v) return s.ok() ? absl::InternalError(absl::StrFormat("rank %d failed to join multicast", r)) : s;
    }
    int32_t bound = 1;
    if (member) {
      s = bind(me, my_slot);
      if (s.ok()) s = map_va({ctx->ranks[me].ordinal}, &mc->va[me]);
      bound = s.ok() ? 1 : 0;
    }
    xs = Exchange(ctx, &bound, sizeof(bound), &all);
    if (!xs.ok()) return xs;
    for (int r = 0; r < ctx->world; ++r) {
      int32_t v;
      std::memcpy(&v, all.data() + r * sizeof(int32_t), sizeof(v));
      if (!v) return s.ok() ? absl::InternalError(absl::StrFormat("rank %d failed to bind multicast", r)) : s;
    }
  }
  {
    absl::Status chk = NvlsSelfCheck(ctx, mc.get(), slots, ctx->self_rank < 0 ? &LocalBarrier : &ExchangeBarrier);
    if (!chk.ok()) return chk;
  }
  guard.armed = false;  // success: the context owns the group (DestroyContext releases it)
  *index = static_cast<int>(ctx->mc_index.size());
  ctx->mc_index.push_back(mc.get());
  ctx->mc_groups[slots] = std::move(mc);
  return absl::OkStatus();
}

}  // namespace rs
