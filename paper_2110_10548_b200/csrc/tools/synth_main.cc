// `synth` — the planner CLI, flag-compatible with the reference tool
// (/root/reference/proj/tools/synth_main.cc:41-59): --system --axes --reduce
// --algo --bytes --size-limit --out --format --seed-order. Without --execute
// the output is byte-identical to the reference's.
//
// --execute [--gpus ORDINALS] [--dtype bf16|f32|i32] [--iters N] runs every
// synthesized program on B200s through redsynth::GpuExecutor (the C-ABI) on
// buffers of --bytes per device and adds measured columns to the JSON report:
// per program "measured_us", "bus_GBps" (nccl-tests AllReduce convention over
// the reduction group), "measured_rank" and "calibrated_us" (B200 cost model,
// rs_plan_predict_us), per matrix "measured_best" and "calibrated_best"
// (SURVEY §8(f) items 3-4). --gpus maps physical device d to CUDA ordinal gpus[d]
// (default: every device on GPU 0 = local mode).
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include <fstream>

#include "nlohmann/json.hpp"
#include "redsynth/executor.h"
#include "redsynth/hierarchy.h"
#include "redsynth/placement.h"
#include "redsynth/report.h"
#include "redsynth/simulator.h"
#include "redsynth/synthesizer.h"
#include "redsynth/topology.h"

namespace {

bool ParseIntList(const std::string& text, std::vector<int>* out) {
  out->clear();
  size_t start = 0;
  while (start <= text.size()) {
    const size_t comma = text.find(',', start);
    const std::string piece = text.substr(start, comma == std::string::npos ? std::string::npos : comma - start);
    char* end = nullptr;
    const long v = std::strtol(piece.c_str(), &end, 10);
    if (piece.empty() || *end != '\0') return false;
    out->push_back(static_cast<int>(v));
    if (comma == std::string::npos) break;
    start = comma + 1;
  }
  return true;
}

int Usage(const char* why) {
  std::cerr << "synth: " << why << "\n"
            << "usage: synth --system PATH --axes LIST --reduce LIST --bytes N "
               "[--algo ring|tree] [--size-limit N] [--out PATH] [--format json|csv] "
               "[--seed-order] [--execute [--gpus LIST] [--dtype bf16|f32|i32] [--iters N]]\n";
  return 2;
}

// Runs every program of the report on the GPUs and returns the augmented JSON.
int Execute(const redsynth::RunRequest& request, const redsynth::Report& report,
            const std::vector<int>& gpus_in, const std::string& dtype_name, int iters, std::string* out) {
  auto system = redsynth::LoadSystemFile(request.system_path);
  if (!system.ok()) return Usage("cannot reload --system");
  const int K = system->device_count();
  std::vector<int> gpus = gpus_in.empty() ? std::vector<int>(K, 0) : gpus_in;
  if (static_cast<int>(gpus.size()) != K) return Usage("--gpus needs one CUDA ordinal per device");
  redsynth::ElementType type = redsynth::ElementType::kBFloat16;
  size_t es = 2;
  if (dtype_name == "f32") {
    type = redsynth::ElementType::kFloat32;
    es = 4;
  } else if (dtype_name == "i32") {
    type = redsynth::ElementType::kInt32;
    es = 4;
  } else if (dtype_name != "bf16") {
    return Usage("--dtype must be bf16, f32 or i32");
  }
  const size_t bytes = static_cast<size_t>(request.payload_bytes);
  const size_t elems = bytes / es;
  auto gpu = redsynth::GpuExecutor::Create(gpus, bytes);
  if (!gpu.ok()) {
    std::cerr << "synth: --execute: " << gpu.status().message() << "\n";
    return 1;
  }
  redsynth::ParallelismSpec spec{request.axes, request.reduction_axes};
  auto matrices = redsynth::EnumerateMatrices(*system, spec);
  if (!matrices.ok()) return 1;
  nlohmann::ordered_json doc = nlohmann::ordered_json::parse(redsynth::ReportToJson(report));
  for (size_t mi = 0; mi < matrices->size(); ++mi) {
    redsynth::SynthesisConfig cfg;
    cfg.size_limit = request.size_limit;
    auto synthesis = redsynth::Synthesize((*matrices)[mi], request.reduction_axes, *system, cfg);
    if (!synthesis.ok()) return 1;
    const auto partition =
        redsynth::ReductionGroupPartition((*matrices)[mi], request.reduction_axes, *system);
    const double n = static_cast<double>(partition.empty() ? 1 : partition[0].size());
    std::vector<double> us(synthesis->programs.size(), 0.0);
    std::vector<double> cal(synthesis->programs.size(), 0.0);
    // Calibrated-model constants: launch latency 3 us when every
    // slot shares one GPU, 8 us across GPUs; 650 GB/s link, 5,967 GB/s HBM.
    const bool one_gpu = std::all_of(gpus.begin(), gpus.end(), [&](int o) { return o == gpus[0]; });
    const double launch_us = one_gpu ? 3.0 : 8.0;
    for (size_t p = 0; p < synthesis->programs.size(); ++p) {
      auto compiled = (*gpu)->Compile(synthesis->programs[p].lowered, elems, type);
      if (!compiled.ok()) {
        std::cerr << "synth: --execute: " << compiled.status().message() << "\n";
        return 1;
      }
      auto t = (*compiled)->TimeUs(1, iters);
      if (!t.ok()) {
        std::cerr << "synth: --execute: " << t.status().message() << "\n";
        return 1;
      }
      us[p] = *t;
      auto c = (*compiled)->PredictUs(launch_us, 650.0, 5967.0);
      if (c.ok()) cal[p] = *c;
    }
    // Measured rank (stable on ties, like RankPrograms).
    std::vector<size_t> order(us.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = i;
    std::stable_sort(order.begin(), order.end(), [&](size_t a, size_t b) { return us[a] < us[b]; });
    std::vector<int> rank_of(us.size());
    for (size_t r = 0; r < order.size(); ++r) rank_of[order[r]] = static_cast<int>(r + 1);
    auto& section = doc["matrices"][mi];
    for (auto& prog : section["programs"]) {
      const int id = prog["id"].get<int>();
      prog["measured_us"] = us[id];
      prog["bus_GBps"] = static_cast<double>(bytes) / (us[id] * 1e-6) * 2.0 * (n - 1.0) / n / 1e9;
      prog["measured_rank"] = rank_of[id];
      prog["calibrated_us"] = cal[id];
    }
    if (!order.empty()) {
      section["measured_best"] = {{"program", static_cast<int>(order[0])}, {"us", us[order[0]]}};
      const size_t cb = static_cast<size_t>(std::min_element(cal.begin(), cal.end()) - cal.begin());
      section["calibrated_best"] = {{"program", static_cast<int>(cb)}, {"measured_us", us[cb]}};
    }
  }
  doc["executed"] = {{"gpus", gpus}, {"dtype", dtype_name}, {"iters", iters},
                     {"executor", "redsynth-b200 sm_100a (C-ABI)"}};
  *out = doc.dump(2) + "\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> flags;
  bool execute = false;
  for (int i = 1; i < argc; ++i) {
    std::string arg = argv[i];
    if (arg == "-h" || arg == "--help") {
      Usage("help");
      return 0;
    }
    if (arg == "--seed-order") continue;  // reserved, no effect (as in the reference)
    if (arg == "--execute") {
      execute = true;
      continue;
    }
    std::string value;
    const size_t eq = arg.find('=');
    if (eq != std::string::npos) {
      value = arg.substr(eq + 1);
      arg = arg.substr(0, eq);
    } else if (i + 1 < argc) {
      value = argv[++i];
    } else {
      return Usage(("missing value for " + arg).c_str());
    }
    static const char* kKnown[] = {"--system", "--axes", "--reduce", "--algo", "--bytes", "--size-limit",
                                   "--out", "--format", "--gpus", "--dtype", "--iters"};
    bool known = false;
    for (const char* k : kKnown) known = known || arg == k;
    if (!known) return Usage(("unknown flag " + arg).c_str());
    flags[arg] = value;
  }
  for (const char* req : {"--system", "--axes", "--reduce", "--bytes"}) {
    if (!flags.count(req)) return Usage((std::string(req) + " is required").c_str());
  }

  redsynth::RunRequest request;
  request.system_path = flags["--system"];
  if (!ParseIntList(flags["--axes"], &request.axes)) return Usage("bad --axes");
  if (!ParseIntList(flags["--reduce"], &request.reduction_axes)) return Usage("bad --reduce");
  char* end = nullptr;
  request.payload_bytes = std::strtoll(flags["--bytes"].c_str(), &end, 10);
  if (*end != '\0') return Usage("bad --bytes");
  if (flags.count("--algo")) {
    const std::string& a = flags["--algo"];
    if (a != "ring" && a != "tree") return Usage("--algo must be ring or tree");
    request.algo = a == "tree" ? redsynth::CollectiveAlgo::kTree : redsynth::CollectiveAlgo::kRing;
  }
  if (flags.count("--size-limit")) request.size_limit = std::atoi(flags["--size-limit"].c_str());
  if (flags.count("--out")) request.out_path = flags["--out"];
  if (flags.count("--format")) {
    const std::string& f = flags["--format"];
    if (f != "json" && f != "csv") return Usage("--format must be json or csv");
    request.format = f == "csv" ? redsynth::ReportFormat::kCsv : redsynth::ReportFormat::kJson;
  }
  if (!execute) {
    const absl::Status status = redsynth::Run(request);
    if (!status.ok()) {
      std::cerr << "synth: " << status.message() << "\n";
      return 1;
    }
    return 0;
  }
  if (request.format != redsynth::ReportFormat::kJson) return Usage("--execute writes JSON only");
  auto report = redsynth::RunPipeline(request);
  if (!report.ok()) {
    std::cerr << "synth: " << report.status().message() << "\n";
    return 1;
  }
  std::vector<int> gpus;
  if (flags.count("--gpus") && !ParseIntList(flags["--gpus"], &gpus)) return Usage("bad --gpus");
  const int iters = flags.count("--iters") ? std::max(1, std::atoi(flags["--iters"].c_str())) : 5;
  std::string text;
  const int rc = Execute(request, *report, gpus, flags.count("--dtype") ? flags["--dtype"] : "bf16", iters, &text);
  if (rc != 0) return rc;
  if (request.out_path.empty()) {
    std::cout << text;
  } else {
    std::ofstream out(request.out_path, std::ios::binary);
    if (!out) return Usage("cannot write --out");
    out << text;
  }
  return 0;
}
