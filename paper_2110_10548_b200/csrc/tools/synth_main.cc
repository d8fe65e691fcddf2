// `synth` — the planner CLI, flag-compatible with the reference tool
// (/root/reference/proj/tools/synth_main.cc:41-59): --system --axes --reduce
// --algo --bytes --size-limit --out --format --seed-order. Own argument
// parser (the reference vendors CLI11, which this repository does not use).
#include <cstdint>
#include <cstdlib>
#include <iostream>
#include <map>
#include <string>
#include <vector>

#include "redsynth/report.h"
#include "redsynth/simulator.h"

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
               "[--seed-order]\n";
  return 2;
}

}  // namespace

int main(int argc, char** argv) {
  std::map<std::string, std::string> flags;
  bool seed_order = false;
  for (int i = 1; i < argc; ++i) {
    std::string arg = argv[i];
    if (arg == "-h" || arg == "--help") return Usage("help"), 0;
    if (arg == "--seed-order") {
      seed_order = true;  // reserved, no effect (as in the reference)
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
    static const char* kKnown[] = {"--system", "--axes", "--reduce", "--algo", "--bytes",
                                   "--size-limit", "--out", "--format"};
    bool known = false;
    for (const char* k : kKnown) known = known || arg == k;
    if (!known) return Usage(("unknown flag " + arg).c_str());
    flags[arg] = value;
  }
  (void)seed_order;
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
  const absl::Status status = redsynth::Run(request);
  if (!status.ok()) {
    std::cerr << "synth: " << status.message() << "\n";
    return 1;
  }
  return 0;
}
