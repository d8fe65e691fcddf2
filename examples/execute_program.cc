// End-to-end C++ host example: the reference planner API (EnumerateMatrices,
// Synthesize) feeding the B200 executor (redsynth::GpuExecutor). Runs every
// synthesized program of a request on int32 data and checks the exact
// identity "device i = sum of its reduction group's inputs".
//   execute_example <system.json> <axes,...> <reduce,...> <elems> [ordinal,...]
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "redsynth/executor.h"
#include "redsynth/hierarchy.h"
#include "redsynth/placement.h"
#include "redsynth/synthesizer.h"
#include "redsynth/topology.h"

static std::vector<int> Ints(const char* s) {
  std::vector<int> v;
  for (const char* p = s; *p;) {
    v.push_back(std::atoi(p));
    while (*p && *p != ',') ++p;
    if (*p == ',') ++p;
  }
  return v;
}

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s system.json axes reduce elems [ordinals]\n", argv[0]);
    return 2;
  }
  auto system = redsynth::LoadSystemFile(argv[1]);
  if (!system.ok()) return std::fprintf(stderr, "%s\n", std::string(system.status().message()).c_str()), 1;
  redsynth::ParallelismSpec spec{Ints(argv[2]), Ints(argv[3])};
  const size_t elems = std::strtoull(argv[4], nullptr, 10);
  const int K = system->device_count();
  std::vector<int> ordinals = argc > 5 ? Ints(argv[5]) : std::vector<int>(K, 0);
  auto gpu = redsynth::GpuExecutor::Create(ordinals, elems * sizeof(int32_t));
  if (!gpu.ok()) return std::fprintf(stderr, "%s\n", std::string(gpu.status().message()).c_str()), 1;
  auto matrices = redsynth::EnumerateMatrices(*system, spec);
  if (!matrices.ok()) return 1;
  int programs = 0, failures = 0;
  std::vector<std::vector<int32_t>> input(K, std::vector<int32_t>(elems));
  for (int d = 0; d < K; ++d)
    for (size_t i = 0; i < elems; ++i) input[d][i] = static_cast<int32_t>((d + 1) * 1000003u + i * 7919u) % 2000000 - 1000000;
  for (const auto& matrix : *matrices) {
    auto synthesis = redsynth::Synthesize(matrix, spec.reduction_axes, *system);
    if (!synthesis.ok()) return 1;
    const auto partition = redsynth::ReductionGroupPartition(matrix, spec.reduction_axes, *system);
    for (const auto& p : synthesis->programs) {
      for (int d = 0; d < K; ++d) {
        void* buf = *(*gpu)->SlotBuffer(d);
        cudaMemcpy(buf, input[d].data(), elems * sizeof(int32_t), cudaMemcpyHostToDevice);
      }
      redsynth::StepFailure failure;
      absl::Status s = (*gpu)->Execute(p.lowered, elems, redsynth::ElementType::kInt32, &failure);
      if (!s.ok()) {
        std::fprintf(stderr, "execute failed: %s\n", std::string(s.message()).c_str());
        return 1;
      }
      ++programs;
      for (const auto& group : partition) {
        std::vector<int32_t> want(elems, 0);
        for (int d : group)
          for (size_t i = 0; i < elems; ++i) want[i] = static_cast<int32_t>(static_cast<uint32_t>(want[i]) + static_cast<uint32_t>(input[d][i]));
        for (int d : group) {
          std::vector<int32_t> got(elems);
          cudaMemcpy(got.data(), *(*gpu)->SlotBuffer(d), elems * sizeof(int32_t), cudaMemcpyDeviceToHost);
          if (std::memcmp(got.data(), want.data(), elems * sizeof(int32_t)) != 0) ++failures;
        }
      }
    }
  }
  // A refused program reports exactly what RunLowered reports.
  redsynth::LoweredProgram bad;
  bad.steps.push_back({{{0, 1}}, redsynth::Collective::kReduce});
  bad.steps.push_back({{{0, 1}}, redsynth::Collective::kReduce});
  redsynth::StepFailure f;
  absl::Status s = (*gpu)->Execute(bad, elems, redsynth::ElementType::kInt32, &f);
  std::printf("programs=%d mismatches=%d refusal='%s' step=%d\n", programs, failures,
              std::string(s.message()).c_str(), f.step);
  return failures == 0 && !s.ok() && f.step == 1 ? 0 : 1;
}
