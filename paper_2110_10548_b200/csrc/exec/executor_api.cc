// redsynth::GpuExecutor — C++ convenience layer over the C-ABI
// (include/redsynth/executor.h). Host-only code; all device work goes
// through rs_plan_run.
#include "redsynth/executor.h"

#include <vector>

#include "redsynth_exec.h"

namespace redsynth {
namespace {

absl::Status FromCode(int code) {
  if (code == RS_OK) return absl::OkStatus();
  return absl::Status(static_cast<absl::StatusCode>(code), rs_last_error());
}

struct Csr {
  std::vector<int32_t> ops, step_ptr, group_ptr, members;
};

Csr ToCsr(const LoweredProgram& lowered) {
  Csr c;
  c.step_ptr.push_back(0);
  c.group_ptr.push_back(0);
  for (const CollectiveStep& step : lowered.steps) {
    c.ops.push_back(static_cast<int32_t>(step.op));
    for (const std::vector<int>& g : step.groups) {
      c.members.insert(c.members.end(), g.begin(), g.end());
      c.group_ptr.push_back(static_cast<int32_t>(c.members.size()));
    }
    c.step_ptr.push_back(static_cast<int32_t>(c.group_ptr.size()) - 1);
  }
  if (c.ops.empty()) c.ops.push_back(0);
  if (c.members.empty()) c.members.push_back(0);
  return c;
}

}  // namespace

CompiledProgram::~CompiledProgram() { rs_plan_destroy(plan_); }

absl::Status CompiledProgram::Run() { return FromCode(rs_plan_run(plan_, nullptr, nullptr)); }

absl::Status CompiledProgram::Run(std::span<void* const> device_buffers) {
  return FromCode(rs_plan_run(plan_, device_buffers.data(), nullptr));
}

absl::StatusOr<double> CompiledProgram::TimeUs(int warmup, int iters) {
  double us = 0;
  absl::Status s = FromCode(rs_plan_time(plan_, warmup, iters, &us));
  if (!s.ok()) return s;
  return us;
}

absl::StatusOr<double> CompiledProgram::PredictUs(double launch_us, double link_gbs, double hbm_gbs) const {
  double us = 0;
  absl::Status s = FromCode(rs_plan_predict_us(plan_, launch_us, link_gbs, hbm_gbs, &us));
  if (!s.ok()) return s;
  return us;
}

int CompiledProgram::launches_per_run() const {
  int n = 0;
  rs_plan_launch_count(plan_, &n);
  return n;
}

absl::StatusOr<std::unique_ptr<GpuExecutor>> GpuExecutor::Create(std::span<const int> cuda_ordinals,
                                                                  size_t max_bytes) {
  rs_ctx* ctx = nullptr;
  const int k = static_cast<int>(cuda_ordinals.size());
  absl::Status s = FromCode(rs_ctx_create(k, cuda_ordinals.data(), max_bytes, &ctx));
  if (!s.ok()) return s;
  return std::unique_ptr<GpuExecutor>(new GpuExecutor(ctx, k));
}

GpuExecutor::~GpuExecutor() { rs_ctx_destroy(ctx_); }

absl::StatusOr<void*> GpuExecutor::SlotBuffer(int slot) const {
  void* p = nullptr;
  absl::Status s = FromCode(rs_ctx_buffer(ctx_, slot, &p));
  if (!s.ok()) return s;
  return p;
}

absl::StatusOr<std::unique_ptr<CompiledProgram>> GpuExecutor::Compile(
    const LoweredProgram& lowered, size_t elems_per_device, ElementType type, StepFailure* failure) {
  // Same verdict and details as the reference's symbolic executor.
  absl::StatusOr<StateContext> symbolic = RunLowered(lowered, k_, failure);
  if (!symbolic.ok()) return symbolic.status();
  const Csr c = ToCsr(lowered);
  rs_plan* plan = nullptr;
  absl::Status s = FromCode(rs_plan_compile(ctx_, static_cast<int>(lowered.steps.size()), c.ops.data(),
                                            c.step_ptr.data(), c.group_ptr.data(), c.members.data(),
                                            elems_per_device, static_cast<int>(type), &plan));
  if (!s.ok()) return s;
  return std::unique_ptr<CompiledProgram>(new CompiledProgram(plan));
}

absl::Status GpuExecutor::Execute(const LoweredProgram& lowered, size_t elems_per_device,
                                  ElementType type, StepFailure* failure) {
  absl::StatusOr<std::unique_ptr<CompiledProgram>> program =
      Compile(lowered, elems_per_device, type, failure);
  if (!program.ok()) return program.status();
  absl::Status s = (*program)->Run();
  if (!s.ok()) return s;
  return Synchronize();
}

absl::Status GpuExecutor::Synchronize() { return FromCode(rs_ctx_synchronize(ctx_)); }

}  // namespace redsynth
