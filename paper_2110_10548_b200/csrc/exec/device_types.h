// Shared host/device launch records of the step kernel.
#ifndef REDSYNTH_B200_EXEC_DEVICE_TYPES_H_
#define REDSYNTH_B200_EXEC_DEVICE_TYPES_H_

#include <cstdint>

#include <cuda_runtime.h>

#include "redsynth_exec.h"

namespace rs {

// One contiguous byte range [lo, hi) (identical offsets in every slot buffer)
// that one owner rank produces: dst_j[x] = src_0[x] + src_1[x] + ... for every
// destination j (sum in source order; a single source is a raw copy).
// Vector tasks are 16-byte aligned at both ends; scalar tasks are the < 16 B
// heads/tails of unaligned ranges.
struct Task {
  uint64_t lo;
  uint64_t hi;
  uint32_t piece_begin;  // first piece of this task within its launch
  uint32_t ptr_begin;    // srcs = ptrs[ptr_begin, +nsrc), dsts follow
  uint16_t nsrc;
  uint16_t ndst;
  uint16_t vec;
  uint16_t mode;  // kModeSum, or kModeNvlsAllReduce: ptrs[ptr_begin] is a multicast
                  // base; dst = multimem.ld_reduce(src) written back with multimem.st
};

constexpr uint16_t kModeSum = 0;
constexpr uint16_t kModeNvlsAllReduce = 1;
// One-shot (LL) task over [lo, hi): pointers tagged with bit 0 are LL packet
// streams (biased: the packet of byte x at +2x, plus the epoch's parity
// region). Untagged sources are local slot buffers (at most one: `local`).
// Tagged destinations receive `local` as packets (sends); untagged
// destinations receive the sum of the sources in order (tagged sources are
// waited for by flag). Whole 8-byte packets cover [lo & ~7, round8(hi)).
constexpr uint16_t kModeLL = 2;
// Push variant: kModeFlagSend copies src -> dst (owner's memory) one
// kFlagChunk piece at a time and then sets that chunk's flag (the pointer
// after dst) to the epoch; kModeFlagRecv sums its sources like kModeSum after
// waiting, per chunk, for each source's flag (nsrc pointers after the dsts,
// null = local source, no wait).
constexpr uint16_t kModeFlagSend = 3;
constexpr uint16_t kModeFlagRecv = 4;
// NVLS Reduce: ptrs[ptr_begin] is a multicast base; multimem.ld_reduce of
// the task's range is stored (unicast) to the ndst destinations that follow.
constexpr uint16_t kModeNvlsReduce = 5;
// NVLS Broadcast: ptrs[ptr_begin] is the root's (local) buffer, ptrs[ptr_begin
// + 1] a multicast base; the root's bytes are stored once to the multicast
// address and the switch writes them into every member (bit copy).
constexpr uint16_t kModeNvlsBroadcast = 6;

// Everything one rank's kernel for one step needs (passed by value).
struct StepArgs {
  const Task* tasks;
  void* const* ptrs;            // slot buffer bases as seen by this rank
  uint32_t ntasks;
  uint32_t npieces;
  uint32_t piece_bytes;         // bytes per vector piece = threads * unroll * 16
  int32_t dtype;
  unsigned int* arrive_counter;  // this rank's CTA-arrival counter
  unsigned int* piece_counter;   // [0] next piece, [1] CTAs done (dynamic push phases)
  uint32_t dynamic;              // 0 static grid stride; pieces from piece_counter: 1 one atomic per piece, 2 next piece reserved ahead
  int* error_flag;               // set to 1 on a barrier timeout
  const uint64_t* inbox;         // this rank's flags, inbox[q] = last epoch of rank q
  uint64_t* signal_ptrs[RS_MAX_RANKS];  // &inbox_of_rank_q[my_rank], every other rank q
  uint32_t nsignal;
  uint32_t nwait;
  uint32_t nfinal;
  uint32_t has_nvls;  // any multimem task: order unicast/multicast aliases (fence.proxy.alias)
  uint32_t has_ll;    // any one-shot task: launch the LL instantiation
  uint32_t signal_done;  // some peer waits for this step's epoch (else no exit fence)
  uint32_t wait_lag;     // entry waits for base + step - wait_lag (one-shot after one-shot: 1)
  uint8_t wait_ranks[RS_MAX_RANKS];
  uint8_t final_ranks[RS_MAX_RANKS];
  // Epochs are relative to a device-resident run base (so a captured CUDA
  // graph can be replayed): step s waits for base + s, publishes base + s + 1;
  // step 0 first publishes base ("inputs in place"); the last step waits the
  // tail barrier for base + num_steps and then advances base by num_steps + 1.
  uint64_t* epoch_base;
  uint32_t step;
  uint32_t num_steps;
  uint64_t timeout_ns;
  uint64_t ll_parity_stride;  // bytes between the two parity regions of an LL block
  uint32_t flag_chunk;        // push-variant chunk (bytes per flag)
  uint32_t recv_piece;        // push reducing piece (divides flag_chunk)
  uint32_t local_only;        // single-rank context: sources are read-only for the launch (.nc loads)
  uint32_t wide_loads;        // cross-GPU pull sums load every source before adding (VectorChunkWide)
  uint32_t pdl;               // launched with programmatic stream serialization
  uint32_t local_wide;        // one-GPU sums load every source before adding
  uint32_t vec256;            // one-GPU bodies move 256-bit vectors
  uint32_t remote256;         // cross-GPU sums move 256-bit vectors
  uint64_t slot_limit;        // bytes addressable per slot region (checked builds assert task ranges)
  uint32_t solo;              // profiling builds only (RS_PROFILING_AIDS): skip every cross-GPU wait
  uint64_t* trace;            // profiling builds only: %globaltimer stamps per piece (RS_TRACE_PTR)
};

// Vector work is cut into pieces of kPieceBytes; a CTA walks a piece in
// chunks of threads * unroll * 16 bytes.
constexpr uint32_t kPieceBytes = 64u << 10;
// LL pieces: 8 packets (64 payload bytes) per thread of a 512-thread CTA,
// all in flight at once.
constexpr uint32_t kLLPieceBytes = 32u << 10;
// Default push-variant chunk (one flag each); also the piece size of
// flagged tasks (Context::flag_chunk, StepArgs::flag_chunk).
constexpr uint32_t kFlagChunk = 256u << 10;  // measured: 64 KiB -3 %, 1 MiB -3 % at K=2

cudaError_t LaunchStep(const StepArgs& args, int grid, int block, int unroll, cudaStream_t stream);

// Emulated ranks: one cooperative launch runs every rank's share of a phase;
// CTAs [prefix[r], prefix[r+1]) are rank r's grid (args[r]).
struct EmulatedArgs {
  StepArgs args[RS_MAX_RANKS];
  uint32_t prefix[RS_MAX_RANKS + 1];
  uint32_t nranks;
};
cudaError_t LaunchEmulated(const EmulatedArgs& e, bool ll, int block, cudaStream_t stream);
int EmulatedResidentCtas(int dtype, int threads, bool ll);  // per SM
// f32 multimem.ld_reduce + multimem.st over [lo, hi) of a multicast VA.
cudaError_t LaunchNvlsSelfCheck(char* mc, uint64_t lo, uint64_t hi, cudaStream_t stream);

}  // namespace rs

#endif  // REDSYNTH_B200_EXEC_DEVICE_TYPES_H_
