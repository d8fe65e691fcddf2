// Host-side executor objects behind the C-ABI (redsynth_exec.h).
#ifndef REDSYNTH_B200_EXEC_INTERNAL_H_
#define REDSYNTH_B200_EXEC_INTERNAL_H_

#include <cstdint>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "absl/status/status.h"
#include "device_types.h"
#include "vmm.h"
#include "redsynth_exec.h"

namespace rs {

// Heap layout of every rank (one cudaMalloc per rank, shared by IPC):
//   [0, 64)        inbox: uint64 epoch per peer rank (written remotely)
//   [256, 260)     CTA-arrival counter
//   [320, 328)     piece queue: next piece, CTAs done (push phases)
//   [512, 516)     barrier-timeout error flag
//   [768, 776)     run base epoch (device resident, starts at 1)
//   [2 MiB, ...)   per hosted slot: its buffer, then `scratch_regions`
//                  scratch buffers (landing zones of the push variant), each
//                  slot_stride bytes (max_bytes rounded up to 2 MiB)
//   then           the one-shot (LL) receive area when world > 1: per sender
//                  rank, two parity regions of 2 * ll_capacity bytes (16-byte
//                  packets {data0, flag, data1, flag} carry 8 payload bytes)
//   then           push-variant chunk flags when world > 1: one uint64 per
//                  flag_chunk (default kFlagChunk = 256 KiB) of every hosted
//                  slot buffer and scratch region
constexpr size_t kInboxOffset = 0;
constexpr size_t kCounterOffset = 256;
constexpr size_t kPieceCounterOffset = 320;  // [320, 328): piece queue of push phases
constexpr size_t kErrorOffset = 512;
constexpr size_t kEpochOffset = 768;
constexpr size_t kDataOffset = 2u << 20;  // multicast-bind granularity
constexpr size_t kSlotAlign = 1 << 21;
// Planning-only contexts and peers driven by other processes: SM count used
// to size pieces when the device attribute is not at hand (B200).
constexpr int kDefaultSmCount = 148;

struct Rank {
  int ordinal = -1;         // CUDA device (meaningful for ranks driven here)
  bool driven = false;      // launched by this process
  char* heap = nullptr;     // local device pointer (driven ranks)
  size_t heap_bytes = 0;
  cudaStream_t stream = nullptr;
  std::vector<char*> view;  // view[q] = rank q's heap as addressed from this rank
  int sm_count = 0;
  VmmBlock vmm;                   // heap allocation when ctx->use_vmm
  std::vector<VmmBlock> imported;  // peers' heaps mapped here (multi-process VMM)
};

// An NVLink multicast object over the slot buffers of one group (one slot per
// GPU), addressed by multimem.ld_reduce / multimem.st.
struct McGroup {
  std::vector<int> slots;
  CUmemGenericAllocationHandle handle = 0;
  size_t bytes = 0;
  std::vector<CUdeviceptr> va;  // per rank: the multicast VA mapped for it (0 = none)
};

typedef int (*ExchangeFn)(const void* send, size_t bytes, void* recv, void* user);

// A pointer-table entry: slot `slot`'s buffer (region -1) or its scratch
// region `region`.
enum { kReduceAuto = -1, kReducePull = 0, kReducePush = 1, kReduceNvls = 2, kReduceNvlsRoot = 3,
       kReducePushRootPulled = 4 };
constexpr int kMcRegion = -2;  // Ref{mc group index, kMcRegion}: a multicast base
// Ref{source slot, kLLRegion, receiver, sender, off}: packets of the source
// slot's data in the receiver rank's LL area, sender's block, parity-0
// region, biased so that the packet of payload byte x sits at +2x (the kernel
// adds the parity). Tagged with bit 0 in the pointer table.
constexpr int kLLRegion = -3;
// Ref{flag id, kFlagRegion, ll_recv = rank, ll_off = byte offset}: a flag
// block of the push variant in that rank's flag area; kNullRegion: nullptr.
constexpr int kFlagRegion = -4;
constexpr int kNullRegion = -5;
constexpr size_t kMaxMcGroups = 32;  // multicast objects per context (switch resources)

struct Ref {
  int slot;    // slot id, or mc group index for kMcRegion
  int region;  // -1 buffer, >= 0 scratch region, kMcRegion multicast, kLLRegion
  int ll_recv = 0;
  int ll_send = 0;
  int64_t ll_off = 0;
  friend bool operator==(const Ref&, const Ref&) = default;
  friend auto operator<=>(const Ref&, const Ref&) = default;
};

class Context {
 public:
  int K = 0;
  size_t max_bytes = 0;
  size_t slot_stride = 0;
  int scratch_regions = 0;  // per slot; the push variant needs >= group size
  int world = 1;
  int self_rank = -1;  // -1: single process drives every rank
  bool peers_open = false;
  bool is_virtual = false;  // planning only: no CUDA resources (CPU tests)
  // Emulated ranks (validation on one GPU, rs_ctx_create_emulated): every
  // rank has its own heap on the same device and each launch phase runs all
  // ranks' steps as one cooperative launch (co-resident CTAs), so ranks that
  // wait on each other never depend on separate launches being co-scheduled.
  bool emulated = false;
  std::vector<int> slot_rank;      // slot -> rank
  std::vector<int> slot_position;  // slot -> index among its rank's slots
  std::vector<Rank> ranks;
  uint64_t timeout_ns = 20ull * 1000 * 1000 * 1000;
  // Cross-GPU sum/copy groups whose data is at least this many bytes use
  // the push variant (one launch, vector bodies cross NVLink as stores only,
  // chunk flags order landing and reduction, senders rotate their targets);
  // smaller ones the one-pass pull-sum-push variant. Measured crossover
  // ~32 MiB at K=2 and K=4; at K=4 push reaches 661-685 GB/s bus from 128 MiB
  // to 1 GiB vs pull 596-646 and NVLS 588-681 (profiles/r01_sweep_k4_push.txt).
  uint64_t push_min_bytes = 32ull << 20;
  int push_max_gpus = RS_MAX_RANKS;  // RS_PUSH_MAX_GPUS
  // Push waves (option "push_wave_bytes", env RS_PUSH_WAVE_BYTES; 0 = one
  // wave): parts are landed and reduced wave by wave so result traffic
  // overlaps landing traffic.
  uint64_t push_wave_bytes = 0;
  // NVLS: AllReduce groups of >= nvls_min_group slots on distinct GPUs use
  // multimem.ld_reduce + multimem.st through the NVSwitch (needs a VMM heap,
  // RS_NVLS=1 at creation; sums then follow the switch's order: f32/bf16
  // results are within tolerance of the ordered oracle, i32 never uses it).
  bool use_vmm = false;
  bool nvls = false;
  int nvls_min_group = 4;
  // NVLS vs the P2P variants: at n = 4 the push variant is as fast or
  // faster at every size (685 vs 681 GB/s bus at 1 GiB) and bit-exact, so
  // groups of < 8 GPUs never use NVLS by default. Groups of >= 8 GPUs move
  // 1.75 c per GPU with P2P vs 1.125 c with NVLS, so they switch at 16 MiB
  // (not measured: no 8-GPU box this round).
  uint64_t nvls_min_bytes = ~0ull;
  uint64_t nvls_min_bytes_n8 = 16ull << 20;
  // Reduce over >= 3 GPUs (semantics.cc:292-299; the root is group[0]):
  //   kReducePull  non-roots own slices, pull every member's copy, sum in
  //                group order, store to the root (bit-exact; default)
  //   kReducePush  same owners, the members land their copies in the owners'
  //                scratch behind chunk flags (stores only; bit-exact)
  //   kReduceNvls  every member owns a slice: multimem.ld_reduce through the
  //                switch, unicast store to the root (f32/bf16, tolerance)
  //   kReduceNvlsRoot  the root issues multimem.ld_reduce for all of R
  //   kReduceAuto  (default) pull below reduce_push_min_bytes, push with
  //                reduce_wave_bytes waves from there. Measured at K=4 bf16
  //                (profiles/r02_reduce_variants_k4.txt): pull 166 / 613 /
  //                2425 us at 64 MiB / 256 MiB / 1 GiB, push with 4 MiB
  //                waves 194 / 554 / 1942 us.
  int reduce_mode = kReduceAuto;
  // NVLS Broadcast (option "nvls_bcast"): on NVLS contexts, Broadcast groups
  // that pass the NVLS size policy use one multicast store stream from the
  // root instead of the P2P relay.
  bool nvls_bcast = false;  // measured slower at K=4 (profiles/r02_bcast_nvls_k4.txt): opt-in
  uint64_t reduce_push_min_bytes = 128ull << 20;
  uint64_t reduce_wave_bytes = 4ull << 20;
  // Push phases with several waves hand out a wave's reducing pieces after
  // the landing pieces of wave_lag later waves (option "wave_lag", env
  // RS_WAVE_LAG): the flags a reducing piece waits on are then more often
  // already set. K=4 Reduce 256 MiB / 512 MiB / 1 GiB: 525 / 958 / 1826 us at
  // lag 0, 514 / 925 / 1781 at lag 2 (profiles/r02_wave_lag.txt).
  int wave_lag = 2;
  // One-shot (LL) steps: when every cross-GPU group of a step has its members
  // on distinct GPUs, each GPU sends any peer at most ll_max_bytes and at most
  // ll_total_bytes in total (payload; packets double it), the step runs as
  // one kernel in which every owner receives its sources as flagged packets
  // pushed into its own LL area and sums locally: no remote loads, no tail
  // wait (latency-bound sizes). The total cap is what binds: measured at K=4
  // one-shot beats pull for AllReduce only at 4 KiB and for Reduce up to
  // 16 KiB, at K=2 for AllReduce up to 16 KiB (profiles/r02_ll_budget.txt).
  // ll_capacity is fixed at creation (RS_LL_CAPACITY); the caps are run-time
  // options.
  uint64_t ll_capacity = 0;
  uint64_t ll_total_bytes = 16u << 10;
  uint64_t ll_max_bytes = 0;
  std::vector<size_t> ll_offset;  // per rank: its LL area within its heap
  std::vector<size_t> flag_offset;  // per rank: push-variant chunk flags (after the LL area)
  std::vector<uint64_t> flag_bytes;
  uint64_t flag_chunk = kFlagChunk;  // push-variant chunk (RS_FLAG_CHUNK at creation)
  // Push reducing pieces (RS_RECV_PIECE; a divisor of flag_chunk, else the
  // chunk itself): a 64 MiB AllReduce at K=4 has 64 reducing chunks per GPU
  // for 148 CTAs, each storing to 4 destinations — smaller pieces keep every
  // CTA busy in the result phase.
  uint64_t recv_piece_bytes = 64u << 10;
  ExchangeFn exchange = nullptr;  // host all-gather (multi-process NVLS setup)
  void* exchange_user = nullptr;
  std::map<std::vector<int>, std::unique_ptr<McGroup>> mc_groups;

  size_t SlotOffset(int slot, int region) const {
    return kDataOffset +
           (static_cast<size_t>(slot_position[slot]) * (1 + scratch_regions) + 1 + region) * slot_stride;
  }
  std::vector<McGroup*> mc_index;  // Ref{i, kMcRegion} -> group
  uint64_t LLRegionBytes() const { return 2 * ll_capacity; }
  char* RefPtr(int viewer, const Ref& r) const {
    if (r.region == kMcRegion) return reinterpret_cast<char*>(mc_index[r.slot]->va[viewer]);
    if (r.region == kNullRegion) return nullptr;
    if (r.region == kFlagRegion) return ranks[viewer].view[r.ll_recv] + flag_offset[r.ll_recv] + r.ll_off;
    if (r.region == kLLRegion) {
      const uintptr_t p = reinterpret_cast<uintptr_t>(ranks[viewer].view[r.ll_recv]) + ll_offset[r.ll_recv] +
                          static_cast<uintptr_t>(r.ll_send) * 2 * LLRegionBytes() + static_cast<uintptr_t>(r.ll_off);
      return reinterpret_cast<char*>(p | 1u);
    }
    return ranks[viewer].view[slot_rank[r.slot]] + SlotOffset(r.slot, r.region);
  }
  char* SlotPtr(int viewer, int slot) const { return RefPtr(viewer, Ref{slot, -1}); }
  std::vector<int> DrivenRanks() const;
};

// One rank's share of one launch phase.
struct RankStep {
  std::vector<Task> tasks;
  std::vector<Ref> ptr_refs;  // pointer-table entries
  uint32_t npieces = 0;
  uint32_t piece_bytes = kPieceBytes;  // 4 KiB .. 64 KiB, sized to fill the GPU
  uint32_t recv_piece = kFlagChunk;    // push reducing piece (divides flag_chunk)
  uint32_t max_grid = 0;      // 0 = resident capacity (one-shot phases: a few CTAs)
  int remote_peers = 0;       // distinct peer GPUs the tasks address
  std::vector<uint8_t> wait;  // ranks to wait for before the phase
  bool signal_done = true;    // a peer waits for this rank's end-of-phase epoch
  double tx_bytes = 0, rx_bytes = 0, hbm_bytes = 0;
};

class Plan {
 public:
  Context* ctx = nullptr;
  int num_steps = 0;   // program steps
  int dtype = 0;
  size_t elems = 0;
  size_t bytes = 0;    // per slot
  int threads = 512;
  int unroll = 4;      // 4 or 8 vectors in flight per thread per source
  int max_ctas = 0;    // 0 = resident capacity
  int ctas_per_sm = 0;  // resident capacity for (dtype, threads, unroll); 0 = recompute
  uint32_t recv_piece = kFlagChunk;  // effective push reducing piece of this plan
  bool dynamic_pieces = true;
  // Phases without chunk flags take their pieces from a prefetched atomic
  // queue instead of a static grid stride (option "piece_queue", env
  // RS_PIECE_QUEUE): 0 never, 1 phases in which the rank touches only its
  // own HBM (N=1 config 2 2864 -> 3110 GB/s, same DRAM bytes), 2 also pull
  // phases (same-box ABAB: N=2 1818 -> 1843, N=4 2127 -> 2151 GB/s, K=4
  // collectives neutral; emulated 8 ranks on one GPU 1215 -> 1150), -1
  // (default) 1 plus 2's pull phases on up to 4 real GPUs, where measured.
  // Only phases with >= 2 pieces per CTA (profiles/r02_piece_queue.txt).
  int piece_queue = -1;
  // Push phases reserve their next piece ahead too (option "push_prefetch",
  // env RS_PUSH_PREFETCH). Deadlock-free (pieces are still handed out in
  // order, so a CTA holding a reserved landing piece of wave w waits only on
  // landings of an earlier wave) but slower: a CTA blocked on chunk flags
  // holds its reserved landing piece back from the peers waiting for it (K=4
  // 64 MiB AllReduce 165 -> 187 us, N=4 2152 -> 2103 GB/s,
  // profiles/r02_piece_queue.txt). Off.
  bool push_prefetch = false;
  bool pdl = false;  // programmatic dependent launch of every step (option "pdl", env RS_PDL): measured neutral
  // cross-GPU pull sums, push landing copies and push reductions with 256-bit
  // vectors (option "remote256", env RS_REMOTE256): K=4 pull 16-256 MiB
  // AllReduce -2.5 %, ReduceScatter -4 %, Reduce -3 % (profiles/r02_remote256_ab.txt)
  bool remote256 = true;
  int vec256 = 2;  // one-GPU 256-bit vectors: 1 copies, 2 copies and sums (option "vec256", env RS_VEC256)
  bool local_wide = false;  // one-GPU sums: all sources in flight (option "local_wide", env RS_LOCAL_WIDE)
  bool wide_loads = true;  // cross-GPU pull sums: all sources in flight (option "wide_loads", env RS_WIDE_LOADS)
  // Launch phases, one per program step (every variant — pull, push with
  // chunk flags, one-shot, NVLS — runs its step in a single launch).
  std::vector<std::vector<RankStep>> phases;  // [phase][rank]
  std::vector<int> phase_step;                // program step of each phase
  std::vector<uint8_t> phase_ll;              // 1: one-shot (LL) phase
  std::vector<uint8_t> phase_lag;             // 1: entry waits one epoch less (LL after LL)
  std::vector<uint8_t> final_wait_bits;       // per rank: ranks for the tail wait
  // Device copies (per driven rank): all tasks / pointer tables of all phases.
  std::vector<StepArgs> launch_args;  // [phase * world + rank], built with ctas_per_sm
  std::vector<int> launch_grid;
  std::vector<Task*> d_tasks;
  std::vector<void**> d_ptrs;
  std::vector<std::vector<size_t>> task_offset, ptr_offset;  // [rank][phase]

  int num_phases() const { return static_cast<int>(phases.size()); }
  ~Plan();
};

absl::Status CreateContext(int K, const int* ordinals, size_t max_bytes, Context** out);
absl::Status CreateRankContext(int K, const int* slot_rank, int world, int rank, int ordinal,
                               size_t max_bytes, Context** out);
absl::Status CreateVirtualContext(int K, const int* slot_rank, int world, Context** out);
absl::Status CreateEmulatedContext(int K, const int* slot_rank, int world, int ordinal, size_t max_bytes,
                                   Context** out);
absl::Status IpcHandle(Context* ctx, void* out);
absl::Status OpenPeers(Context* ctx, const void* handles);
absl::Status DestroyContext(Context* ctx);
absl::Status Synchronize(Context* ctx);
// Creates (collectively, in multi-process mode) or finds the multicast object
// over `slots`; returns its index for Ref{index, kMcRegion}.
absl::Status EnsureMulticast(Context* ctx, const std::vector<int>& slots, int* index);

absl::Status CompilePlan(Context* ctx, int num_steps, const int32_t* step_op,
                         const int32_t* step_group_ptr, const int32_t* group_member_ptr,
                         const int32_t* members, size_t elems, int dtype, Plan** out);
absl::Status RunPlan(Plan* plan, void* const* device_bufs, void* const* host_bufs,
                     void* const* streams);

std::string DescribePlan(const Plan& plan);
// Launch records (StepArgs + grid) of every (phase, driven rank); called on
// the first run after compilation or a launch-shape change.
void BuildLaunches(Plan* plan);

int MaxResidentCtas(int dtype, int threads, int unroll);  // per SM, from the occupancy API

absl::Status CudaStatus(cudaError_t err, const char* what);

}  // namespace rs

#endif  // REDSYNTH_B200_EXEC_INTERNAL_H_
