// Test-infrastructure C-ABI over the UNMODIFIED reference library
// (oracle/_ref/libredsynth_ref.so). Lets the Python tests and the golden-
// fixture script drive the reference planner and its symbolic executor
// (`RunLowered`, /root/reference/proj/src/dsl.cc:142-164) through ctypes.
// Only tests/, tests/golden/make_golden.py and bench.py's reference arm may
// load this library; it is never on the product path.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "nlohmann/json.hpp"
#include "redsynth/dsl.h"
#include "redsynth/hierarchy.h"
#include "redsynth/placement.h"
#include "redsynth/report.h"
#include "redsynth/semantics.h"
#include "redsynth/simulator.h"
#include "redsynth/synthesizer.h"
#include "redsynth/topology.h"

namespace {

char* Dup(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

redsynth::LoweredProgram FromCsr(int num_steps, const int* ops, const int* step_group_ptr,
                                 const int* group_member_ptr, const int* members) {
  redsynth::LoweredProgram lowered;
  for (int s = 0; s < num_steps; ++s) {
    redsynth::CollectiveStep step;
    step.op = static_cast<redsynth::Collective>(ops[s]);
    for (int g = step_group_ptr[s]; g < step_group_ptr[s + 1]; ++g) {
      step.groups.emplace_back(members + group_member_ptr[g], members + group_member_ptr[g + 1]);
    }
    lowered.steps.push_back(std::move(step));
  }
  return lowered;
}

}  // namespace

extern "C" {

void ref_free(char* p) { std::free(p); }

// Enumerate + synthesize + simulate every placement, return JSON:
// {"device_count":K,"matrices":[{"factors":[[..]],"partition":[[..]],
//   "hierarchy":[labels],"programs":[{"text":..,"seconds":..,
//   "steps":[{"op":i,"groups":[[..]]}]}]}]}   (programs in emission order)
// Returns the absl status code; on error *out holds the message.
int ref_synthesize(const char* system_json, const int* axes, int n_axes, const int* reduce,
                   int n_reduce, int size_limit, long long payload_bytes, int algo,
                   char** out) {
  auto system = redsynth::ParseSystem(system_json);
  if (!system.ok()) {
    *out = Dup(std::string(system.status().message()));
    return static_cast<int>(system.status().code());
  }
  redsynth::ParallelismSpec spec{.axes = std::vector<int>(axes, axes + n_axes),
                                 .reduction_axes = std::vector<int>(reduce, reduce + n_reduce)};
  auto matrices = redsynth::EnumerateMatrices(*system, spec);
  if (!matrices.ok()) {
    *out = Dup(std::string(matrices.status().message()));
    return static_cast<int>(matrices.status().code());
  }
  nlohmann::ordered_json doc;
  doc["device_count"] = system->device_count();
  doc["matrices"] = nlohmann::ordered_json::array();
  for (const auto& matrix : *matrices) {
    nlohmann::ordered_json m;
    std::vector<std::vector<int>> factors;
    for (int a = 0; a < matrix.num_axes(); ++a) factors.push_back(matrix.AxisRow(a));
    m["factors"] = factors;
    m["partition"] =
        redsynth::ReductionGroupPartition(matrix, spec.reduction_axes, *system);
    redsynth::SynthesisConfig cfg{.size_limit = size_limit};
    auto result = redsynth::Synthesize(matrix, spec.reduction_axes, *system, cfg);
    if (!result.ok()) {
      *out = Dup(std::string(result.status().message()));
      return static_cast<int>(result.status().code());
    }
    std::vector<std::string> labels;
    for (const auto& level : result->hierarchy.levels) labels.push_back(level.label);
    m["hierarchy"] = labels;
    m["programs"] = nlohmann::ordered_json::array();
    for (const auto& entry : result->programs) {
      nlohmann::ordered_json p;
      p["text"] = redsynth::PrettyPrint(entry.program, result->hierarchy);
      redsynth::CostModelConfig cost{.algo = algo == 1 ? redsynth::CollectiveAlgo::kTree
                                                       : redsynth::CollectiveAlgo::kRing,
                                     .payload_bytes = payload_bytes};
      auto sim = redsynth::Simulate(entry.lowered, *system, cost);
      p["seconds"] = sim.ok() ? sim->total_seconds : -1.0;
      p["steps"] = nlohmann::ordered_json::array();
      for (const auto& step : entry.lowered.steps) {
        p["steps"].push_back({{"op", static_cast<int>(step.op)}, {"groups", step.groups}});
      }
      m["programs"].push_back(std::move(p));
    }
    doc["matrices"].push_back(std::move(m));
  }
  *out = Dup(doc.dump());
  return 0;
}

// The reference symbolic executor. On success writes the final boolean
// state as k*k*k bytes (device-major, then row, then column) into `state`
// (may be null). On failure returns FAILED_PRECONDITION / INVALID_ARGUMENT
// and fills fail_step / fail_violation (RuleViolation enum) and `msg`.
int ref_run_lowered(int num_steps, const int* ops, const int* step_group_ptr,
                    const int* group_member_ptr, const int* members, int k,
                    unsigned char* state, int* fail_step, int* fail_violation, char* msg,
                    int msg_len) {
  redsynth::LoweredProgram lowered =
      FromCsr(num_steps, ops, step_group_ptr, group_member_ptr, members);
  redsynth::StepFailure failure;
  auto ctx = redsynth::RunLowered(lowered, k, &failure);
  if (!ctx.ok()) {
    if (fail_step) *fail_step = failure.step;
    if (fail_violation) *fail_violation = static_cast<int>(failure.violation);
    if (msg && msg_len > 0) {
      std::string m(ctx.status().message());
      std::strncpy(msg, m.c_str(), msg_len - 1);
      msg[msg_len - 1] = '\0';
    }
    return static_cast<int>(ctx.status().code());
  }
  if (state) {
    for (int d = 0; d < k; ++d)
      for (int r = 0; r < k; ++r)
        for (int c = 0; c < k; ++c)
          state[(static_cast<size_t>(d) * k + r) * k + c] = ctx->state(d).bit(r, c) ? 1 : 0;
  }
  return 0;
}

// Times `iters` executions of RunLowered (the reference CPU "executor"),
// returning mean microseconds per program.
double ref_time_run_lowered(int num_steps, const int* ops, const int* step_group_ptr,
                            const int* group_member_ptr, const int* members, int k, int iters);

// Full pipeline report (ReportToJson / ReportToCsv) for byte comparison.
int ref_report(const char* system_path, const int* axes, int n_axes, const int* reduce,
               int n_reduce, int size_limit, long long payload_bytes, int algo, int csv,
               char** out) {
  redsynth::RunRequest request;
  request.system_path = system_path;
  request.axes.assign(axes, axes + n_axes);
  request.reduction_axes.assign(reduce, reduce + n_reduce);
  request.algo = algo == 1 ? redsynth::CollectiveAlgo::kTree : redsynth::CollectiveAlgo::kRing;
  request.payload_bytes = payload_bytes;
  request.size_limit = size_limit;
  auto report = redsynth::RunPipeline(request);
  if (!report.ok()) {
    *out = Dup(std::string(report.status().message()));
    return static_cast<int>(report.status().code());
  }
  *out = Dup(csv ? redsynth::ReportToCsv(*report) : redsynth::ReportToJson(*report));
  return 0;
}

}  // extern "C"

#include <chrono>

extern "C" double ref_time_run_lowered(int num_steps, const int* ops, const int* step_group_ptr,
                                       const int* group_member_ptr, const int* members, int k,
                                       int iters) {
  redsynth::LoweredProgram lowered =
      FromCsr(num_steps, ops, step_group_ptr, group_member_ptr, members);
  auto t0 = std::chrono::steady_clock::now();
  int ok = 0;
  for (int i = 0; i < iters; ++i) ok += redsynth::RunLowered(lowered, k).ok() ? 1 : 0;
  auto t1 = std::chrono::steady_clock::now();
  if (ok < 0) return -1.0;
  return std::chrono::duration<double, std::micro>(t1 - t0).count() / (iters > 0 ? iters : 1);
}
