// Executor contexts: per-rank heaps (slot buffers + barrier flags), peer
// mappings (CUDA peer access in one process, CUDA IPC across processes) and
// streams.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>

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
  int hosted = 0;
  for (int d = 0; d < ctx->K; ++d) hosted += ctx->slot_rank[d] == r;
  rank.heap_bytes =
      kDataOffset + static_cast<size_t>(hosted) * (1 + ctx->scratch_regions) * ctx->slot_stride;
  void* heap = nullptr;
  RS_CUDA(cudaMalloc(&heap, rank.heap_bytes));
  rank.heap = static_cast<char*>(heap);
  RS_CUDA(cudaMemset(rank.heap, 0, kDataOffset));
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
}

void ReadTimeoutEnv(Context* ctx) {
  if (const char* env = std::getenv("RS_BARRIER_TIMEOUT_S")) {
    const double s = std::atof(env);
    if (s > 0) ctx->timeout_ns = static_cast<uint64_t>(s * 1e9);
  }
  if (const char* env = std::getenv("RS_PUSH_MIN_BYTES")) {
    ctx->push_min_bytes = std::strtoull(env, nullptr, 10);
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
  absl::Status s = AllocateRank(ctx.get(), rank);
  if (!s.ok()) {
    DestroyContext(ctx.release());
    return s;
  }
  ctx->peers_open = world == 1;
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
    cudaIpcMemHandle_t h;
    std::memcpy(&h, bytes + static_cast<size_t>(q) * RS_IPC_HANDLE_BYTES, sizeof(h));
    void* p = nullptr;
    RS_CUDA(cudaIpcOpenMemHandle(&p, h, cudaIpcMemLazyEnablePeerAccess));
    me.view[q] = static_cast<char*>(p);
  }
  ctx->peers_open = true;
  return absl::OkStatus();
}

absl::Status Synchronize(Context* ctx) {
  for (int r : ctx->DrivenRanks()) {
    Rank& rank = ctx->ranks[r];
    RS_CUDA(cudaSetDevice(rank.ordinal));
    RS_CUDA(cudaStreamSynchronize(rank.stream));
    int err = 0;
    RS_CUDA(cudaMemcpy(&err, rank.heap + kErrorOffset, sizeof(int), cudaMemcpyDeviceToHost));
    if (err) {
      return absl::InternalError(absl::StrFormat(
          "rank %d: inter-GPU barrier timed out (a peer never reached the step); results are invalid",
          r));
    }
  }
  return absl::OkStatus();
}

absl::Status DestroyContext(Context* ctx) {
  if (ctx == nullptr) return absl::OkStatus();
  for (int r = 0; r < ctx->world; ++r) {
    Rank& rank = ctx->ranks[r];
    if (!rank.driven) continue;
    cudaSetDevice(rank.ordinal);
    if (rank.stream) cudaStreamSynchronize(rank.stream);
    if (ctx->self_rank >= 0) {
      for (int q = 0; q < ctx->world; ++q)
        if (q != r && rank.view.size() > static_cast<size_t>(q) && rank.view[q]) cudaIpcCloseMemHandle(rank.view[q]);
    }
    if (rank.stream) cudaStreamDestroy(rank.stream);
    if (rank.heap) cudaFree(rank.heap);
  }
  delete ctx;
  return absl::OkStatus();
}

}  // namespace rs
