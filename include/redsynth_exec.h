/* redsynth-b200 executor C-ABI — the drop-in boundary of the hot path.
 *
 * Executes a synthesized reduction program (a LoweredProgram: steps of
 * AllReduce / ReduceScatter / AllGather / Reduce / Broadcast over disjoint
 * device groups) on B200 GPUs with hand-written sm_100a peer-to-peer kernels.
 * It is the data-moving sibling of the reference's symbolic executor
 *
 *   absl::StatusOr<StateContext> RunLowered(const LoweredProgram&, int k,
 *                                           StepFailure* = nullptr);
 *     — /root/reference/proj/include/redsynth/dsl.h:108, src/dsl.cc:142-164
 *
 * and is called by the C++ wrapper redsynth::Execute (redsynth/executor.h),
 * by the Python host mirror (paper_2110_10548_b200/executor.py, ctypes) and by
 * the bench. No torch or C++ types cross this boundary.
 *
 * Vocabulary. K "slots" = the K physical device ids of the program
 * (SystemModel::device_count()). Slot d holds an N-element buffer; row r of it
 * is elements [floor(r*N/K), floor((r+1)*N/K)). Slots live on "ranks" = GPUs.
 * One process may drive all ranks (rs_ctx_create) or one rank each
 * (rs_ctx_create_rank + IPC handle exchange, e.g. over torch.distributed).
 * Several slots may share one GPU (e.g. K = 8 slots on 1 GPU = "local mode":
 * every collective becomes an HBM-local sum/copy).
 *
 * Status codes mirror absl::StatusCode: 0 OK, 3 INVALID_ARGUMENT,
 * 9 FAILED_PRECONDITION (a rule violation, same wording as
 * StepFailure::Describe, dsl.cc:135-140), 13 INTERNAL (CUDA error, a
 * device-side barrier timeout, or a checked-build assertion), 14 UNAVAILABLE
 * (no GPU / extension missing).
 * rs_last_error() returns the message of the last failing call on the thread.
 */
#ifndef REDSYNTH_EXEC_H_
#define REDSYNTH_EXEC_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct rs_ctx rs_ctx;
typedef struct rs_plan rs_plan;

enum { RS_OK = 0, RS_INVALID_ARGUMENT = 3, RS_FAILED_PRECONDITION = 9, RS_INTERNAL = 13,
       RS_UNAVAILABLE = 14 };
/* Element types. */
enum { RS_F32 = 0, RS_BF16 = 1, RS_I32 = 2 };
/* Collective enum order of /root/reference/proj/include/redsynth/semantics.h:29-35. */
enum { RS_OP_ALLREDUCE = 0, RS_OP_REDUCESCATTER = 1, RS_OP_ALLGATHER = 2, RS_OP_REDUCE = 3,
       RS_OP_BROADCAST = 4 };

#define RS_MAX_RANKS 8
#define RS_IPC_HANDLE_BYTES 64

/* Last error message of the calling thread ("" when none). */
const char* rs_last_error(void);
/* Library version string. */
const char* rs_version(void);

/* ---- contexts ----------------------------------------------------------- */

/* Single process drives all K slots. cuda_ordinals[d] = GPU of slot d (the
 * physical-device -> CUDA-ordinal map); repeated ordinals put several slots on
 * one GPU. Each distinct ordinal is one rank. Allocates, per rank, a heap with
 * one max_bytes buffer per hosted slot plus barrier flags, and enables peer
 * access between the ranks. */
int rs_ctx_create(int K, const int* cuda_ordinals, size_t max_bytes, rs_ctx** out);

/* One process per GPU. slot_rank[d] = rank hosting slot d (0..world_size-1);
 * this process is `rank` on GPU `cuda_ordinal`. Follow with
 * rs_ctx_ipc_handle on every rank, an all-gather of the handles, and
 * rs_ctx_open_peers. Every rank must then compile and run the same plans in
 * the same order (like NCCL collectives). */
int rs_ctx_create_rank(int K, const int* slot_rank, int world_size, int rank, int cuda_ordinal,
                       size_t max_bytes, rs_ctx** out);
/* Writes RS_IPC_HANDLE_BYTES bytes identifying this rank's heap. */
int rs_ctx_ipc_handle(rs_ctx* ctx, void* out);
/* handles = world_size * RS_IPC_HANDLE_BYTES bytes, rank-major. */
int rs_ctx_open_peers(rs_ctx* ctx, const void* handles);

/* Validation mode: world_size (2..8) ranks emulated on ONE GPU. Every rank
 * gets its own heap (slot buffers, scratch, flags, one-shot area) on
 * cuda_ordinal, and each launch phase runs every rank's step kernel as ONE
 * cooperative launch, so ranks that wait on each other's flags are
 * co-resident (separate launches on one GPU are not guaranteed to run
 * concurrently). Exercises the cross-rank kernels — pull over "peer"
 * pointers, one-shot packets, push chunk flags, epoch barriers — exactly as
 * compiled for world_size GPUs, without them; not a performance mode, no
 * NVLS. Plans run on the stream of the first local rank. */
int rs_ctx_create_emulated(int K, const int* slot_rank, int world_size, int cuda_ordinal, size_t max_bytes,
                           rs_ctx** out);

/* Planning-only context: no GPU, no memory. Plans compiled on it can be
 * inspected with rs_plan_describe_json but not run (CPU tests, tooling). */
int rs_ctx_create_virtual(int K, const int* slot_rank, int world_size, rs_ctx** out);

int rs_ctx_destroy(rs_ctx* ctx);

/* Device pointer of the executor-owned buffer of slot d (slots hosted by this
 * process only). Programs run in place on these buffers when rs_plan_run is
 * given no user buffers. */
int rs_ctx_buffer(rs_ctx* ctx, int slot, void** device_ptr);
/* Copy `bytes` between host memory (pinned for speed) and the start of slot
 * d's buffer (hosted slots only), asynchronously on `stream` (NULL = the
 * context's stream of that slot's GPU). Used to stage inputs once and run
 * several plans in place before reading the results back. */
int rs_ctx_upload(rs_ctx* ctx, int slot, const void* host, size_t bytes, void* stream);
int rs_ctx_download(rs_ctx* ctx, int slot, void* host, size_t bytes, void* stream);
/* Number of ranks driven by this process and their CUDA ordinals. */
int rs_ctx_local_ranks(rs_ctx* ctx, int* count, int* ordinals /* RS_MAX_RANKS */);
/* Context knobs applied to plans compiled afterwards: "push_min_bytes"
 * (cross-GPU AllReduce / balanced AllGather groups moving at least this many
 * bytes use the push variant: one launch, vector data crosses NVLink as
 * stores only, chunk flags order landing and reduction; -1 disables it;
 * default 32 MiB, env RS_PUSH_MIN_BYTES), "push_wave_bytes" (push parts are
 * landed and reduced in waves of this size; default 0 = one wave) and
 * "barrier_timeout_ms" (device-side spin limit, default 20 s). Scratch
 * for the push variant is reserved at creation: min(K, 8) buffers per slot on
 * multi-GPU contexts (env RS_SCRATCH_REGIONS). "ll_max_bytes" /
 * "ll_total_bytes": a step whose cross-GPU groups have one member per GPU and
 * in which no GPU sends a peer more than ll_max_bytes and no GPU sends more
 * than ll_total_bytes in total runs one-shot (LL): sources are pushed as
 * flagged 16-byte packets into each receiver's LL area and every destination
 * sums locally, in group order (bit-exact like the pull path); 0 disables it
 * (defaults 256 KiB and 16 KiB, env RS_LL_MAX_BYTES / RS_LL_TOTAL_BYTES,
 * capped by the per-peer area reserved at creation, env RS_LL_CAPACITY,
 * default 512 KiB). "reduce_mode" for Reduce over >= 3 GPUs: -1 auto
 * (default: pull below "reduce_push_min_bytes" = 128 MiB, push with
 * "reduce_wave_bytes" = 4 MiB waves above), 0 pull, 1 push, 2 NVLS (members
 * reduce slices through the switch, store to the root; tolerance), 3 NVLS
 * with the root reducing everything, 4 push with the root's copy pulled by
 * the owners (measured slower; kept for A/B). "wave_lag" (default 2): push
 * phases with several waves hand out a wave's reducing pieces after the
 * landing pieces of that many later waves. */
int rs_ctx_set_option(rs_ctx* ctx, const char* key, long long value);

/* NVLS (NVLink SHARP): with RS_NVLS=1 at context creation the heaps are
 * cuMemCreate'd (shared across processes as POSIX fds via pidfd_getfd) and
 * AllReduce groups of >= "nvls_min_group" (default 4) slots on distinct GPUs
 * run as multimem.ld_reduce + multimem.st through the NVSwitch. The switch
 * sums in its own order, so f32/bf16 results match the ordered oracle within
 * tolerance instead of bit for bit (i32 never uses NVLS). Options "nvls"
 * (0/1), "nvls_min_group" and "nvls_min_bytes" (default: never for groups
 * of < 8 GPUs, where the push variant is as fast; 16 MiB for >= 8; env
 * RS_NVLS_MIN_BYTES) tune later compiles. */
int rs_ctx_nvls(rs_ctx* ctx, int* enabled);
/* Host all-gather used to set up multicast objects collectively in the
 * one-process-per-GPU mode: fn(send, bytes, recv[world * bytes], user) must
 * gather `bytes` from every rank in rank order and return 0. Plan compiles
 * are then collective (every rank compiles the same programs in order). */
typedef int (*rs_exchange_fn)(const void* send, size_t bytes, void* recv, void* user);
int rs_ctx_set_exchange(rs_ctx* ctx, rs_exchange_fn fn, void* user);
/* Blocks until all work on the context's GPUs is done (device-wide: plans
 * usually run on caller streams); reports a device-side barrier timeout
 * (INTERNAL) once, then clears it. */
int rs_ctx_synchronize(rs_ctx* ctx);

/* ---- plans -------------------------------------------------------------- */

/* Compiles a lowered program (CSR: step_op[num_steps], step_group_ptr
 * [num_steps+1] into group_member_ptr[num_groups+1] into members[]) for
 * buffers of elems_per_device elements of `dtype`. Refuses programs that
 * RunLowered refuses (same step index and violation), steps whose groups are
 * not disjoint, and sizes above the context's max_bytes. */
int rs_plan_compile(rs_ctx* ctx, int num_steps, const int32_t* step_op,
                    const int32_t* step_group_ptr, const int32_t* group_member_ptr,
                    const int32_t* members, size_t elems_per_device, int dtype, rs_plan** out);

/* Enqueues the program (async). device_bufs: NULL = run in place on the
 * context buffers; else K device pointers indexed by slot (entries of slots
 * not hosted here are ignored) that are copied in before and out after.
 * streams: NULL = the context's own streams; else one cudaStream_t per local
 * rank, in rs_ctx_local_ranks order. */
int rs_plan_run(rs_plan* plan, void* const* device_bufs, void* const* streams);

/* End-to-end variant: host_bufs = K host pointers (pinned for speed) indexed
 * by slot; copies each hosted slot's host buffer in (H2D), runs, copies the
 * result back (D2H). Async on the given/own streams. */
int rs_plan_run_host(rs_plan* plan, void* const* host_bufs, void* const* streams);

/* Device time of one run: `warmup` untimed runs, then `iters` back-to-back
 * runs bracketed by CUDA events on every local rank's stream; *us = the
 * slowest rank's elapsed time / iters. Synchronous. */
int rs_plan_time(rs_plan* plan, int warmup, int iters, double* us);

/* Kernel launches one rs_plan_run performs (all local ranks). */
int rs_plan_launch_count(rs_plan* plan, int* launches);

/* Per-step summary, for reporting: algorithmic bytes each rank moves over
 * links (link_bytes) and through HBM (hbm_bytes) in step s, maxed over ranks. */
int rs_plan_step_bytes(rs_plan* plan, int step, double* link_bytes, double* hbm_bytes);

/* B200-calibrated cost of one run, next to the
 * reference's Simulate (simulator.cc:141-188): per launch phase,
 * launch_us + max over GPUs of link bytes per direction / link_gbs + max over
 * GPUs of HBM bytes / hbm_gbs. Unlike the reference model it sees the
 * executor's actual traffic: per-port non-blocking NVSwitch (no shared-switch
 * division), local steps at HBM speed, relay fan-out, one-shot and NVLS
 * variants. Planning-only contexts work (no GPU needed). */
int rs_plan_predict_us(rs_plan* plan, double launch_us, double link_gbs, double hbm_gbs, double* us);

/* Tuning knobs (0 = default): CTAs per launch cap and threads per CTA. */
int rs_plan_set_launch(rs_plan* plan, int max_ctas, int threads);
/* Named knobs: "unroll" (4|8 vectors in flight per thread per source),
 * "threads" (per CTA), "max_ctas" (per launch, 0 = resident capacity),
 * "wide_loads" (cross-GPU sums load every source before adding; default 1),
 * "dynamic_pieces" (push phases take pieces from an atomic queue; default 1),
 * "pdl" (programmatic dependent launch; default 0, measured neutral),
 * "local_wide" (one-GPU sums load every source first; default 0),
 * "vec256" (one-GPU 256-bit vectors: 0 off, 1 copies, 2 copies and sums;
 * default 2), "remote256" (cross-GPU 256-bit vectors; default 1),
 * "piece_queue" (phases without chunk flags take pieces from a prefetched
 * atomic queue: 0 never, 1 phases touching only the rank's own HBM, 2 also
 * pull phases, -1 (default) 1 plus pull phases on up to 4 real GPUs; only
 * phases with >= 2 pieces per CTA, never NVLS or one-shot phases),
 * "push_prefetch" (push phases reserve their next piece ahead too; default
 * 0, measured slower). */
int rs_plan_set_option(rs_plan* plan, const char* key, long long value);

/* JSON dump of the compiled plan: per step, per rank, the entry-barrier
 * ranks and tasks {lo, hi (bytes), vec, src slots, dst slots}. */
int rs_plan_describe_json(rs_plan* plan, char** out_json);

int rs_plan_destroy(rs_plan* plan);

/* ---- planner (host C++ behind C, for the Python mirror) ------------------ */

/* Runs EnumerateMatrices + Synthesize (+ Simulate for `seconds`) and returns
 * JSON {"device_count", "matrices": [{"factors", "partition", "hierarchy",
 * "programs": [{"text", "seconds", "steps": [{"op", "groups"}]}]}]}.
 * Free with rs_free. */
int rs_synthesize_json(const char* system_json, const int* axes, int n_axes,
                       const int* reduce, int n_reduce, int size_limit, long long payload_bytes,
                       int algo, char** out_json);
/* RunPipeline + ReportToJson/ReportToCsv (byte-identical to the reference). */
int rs_report(const char* system_path, const int* axes, int n_axes, const int* reduce,
              int n_reduce, int size_limit, long long payload_bytes, int algo, int csv,
              char** out);
/* Symbolic RunLowered through the host planner (final state as K*K*K bytes). */
int rs_run_lowered(int num_steps, const int32_t* step_op, const int32_t* step_group_ptr,
                   const int32_t* group_member_ptr, const int32_t* members, int k,
                   unsigned char* state, int* fail_step, int* fail_violation);
void rs_free(char* p);

#ifdef __cplusplus
}
#endif

#endif /* REDSYNTH_EXEC_H_ */
