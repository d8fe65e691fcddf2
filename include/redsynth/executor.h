// redsynth-b200 — GPU executor, the data-moving sibling of RunLowered
// (/root/reference/proj/include/redsynth/dsl.h:108). A thin C++ layer over
// the C-ABI in include/redsynth_exec.h, in the reference's own conventions
// (absl::Status codes, StepFailure details, value types, const refs).
//
//   auto gpu = redsynth::GpuExecutor::Create({0, 0, 1, 1, 2, 2, 3, 3}, 256 << 20);
//   // ... fill (*gpu)->SlotBuffer(d) with each device's data ...
//   redsynth::StepFailure failure;
//   absl::Status s = (*gpu)->Execute(program.lowered, elems, redsynth::ElementType::kBFloat16,
//                                    &failure);   // same refusals as RunLowered
#ifndef REDSYNTH_EXECUTOR_H_
#define REDSYNTH_EXECUTOR_H_

#include <cstddef>
#include <memory>
#include <span>

#include "absl/status/status.h"
#include "absl/status/statusor.h"
#include "redsynth/dsl.h"

struct rs_ctx;
struct rs_plan;

namespace redsynth {

enum class ElementType { kFloat32 = 0, kBFloat16 = 1, kInt32 = 2 };

class GpuExecutor;

// A program compiled for one executor and one buffer size (reusable).
class CompiledProgram {
 public:
  ~CompiledProgram();
  CompiledProgram(const CompiledProgram&) = delete;
  CompiledProgram& operator=(const CompiledProgram&) = delete;

  // Enqueues one execution in place on the executor's slot buffers
  // (asynchronous; GpuExecutor::Synchronize waits and reports barrier errors).
  absl::Status Run();
  // Copies K device buffers (slot-indexed) in, runs, copies them back out.
  absl::Status Run(std::span<void* const> device_buffers);
  int launches_per_run() const;
  // Device time of one run in microseconds (warmup untimed runs, then iters
  // timed back-to-back runs; slowest GPU). Synchronous.
  absl::StatusOr<double> TimeUs(int warmup = 1, int iters = 5);
  // B200-calibrated cost of one run in microseconds from the plan's own
  // traffic (rs_plan_predict_us): per launch, launch_us + link bytes /
  // link_gbs + HBM bytes / hbm_gbs (maxed over GPUs).
  absl::StatusOr<double> PredictUs(double launch_us, double link_gbs, double hbm_gbs) const;

 private:
  friend class GpuExecutor;
  explicit CompiledProgram(rs_plan* plan) : plan_(plan) {}
  rs_plan* plan_;
};

class GpuExecutor {
 public:
  // One process drives every GPU: slot d (= physical device id d of the
  // lowered programs) lives on CUDA device cuda_ordinals[d]; slots may share
  // a GPU. Each slot gets a max_bytes buffer.
  static absl::StatusOr<std::unique_ptr<GpuExecutor>> Create(std::span<const int> cuda_ordinals,
                                                             size_t max_bytes);
  ~GpuExecutor();
  GpuExecutor(const GpuExecutor&) = delete;
  GpuExecutor& operator=(const GpuExecutor&) = delete;

  int device_count() const { return k_; }
  // Device pointer of slot d's buffer.
  absl::StatusOr<void*> SlotBuffer(int slot) const;

  // Validates like RunLowered (same status, same StepFailure) and compiles.
  absl::StatusOr<std::unique_ptr<CompiledProgram>> Compile(const LoweredProgram& lowered,
                                                           size_t elems_per_device,
                                                           ElementType type,
                                                           StepFailure* failure = nullptr);

  // Compile + Run + Synchronize.
  absl::Status Execute(const LoweredProgram& lowered, size_t elems_per_device, ElementType type,
                       StepFailure* failure = nullptr);

  absl::Status Synchronize();

 private:
  GpuExecutor(rs_ctx* ctx, int k) : ctx_(ctx), k_(k) {}
  rs_ctx* ctx_;
  int k_;
};

}  // namespace redsynth

#endif  // REDSYNTH_EXECUTOR_H_
