// extern "C" surface of libredsynth_b200.so (declared in include/redsynth_exec.h).
#include <cstdlib>
#include <cstring>
#include <string>

#include "exec_internal.h"
#include "nlohmann/json.hpp"
#include "redsynth/dsl.h"
#include "redsynth/hierarchy.h"
#include "redsynth/placement.h"
#include "redsynth/report.h"
#include "redsynth/simulator.h"
#include "redsynth/synthesizer.h"
#include "redsynth/topology.h"

struct rs_ctx {
  rs::Context* impl;
};
struct rs_plan {
  rs::Plan* impl;
};

namespace {

thread_local std::string g_last_error;

int Report(const absl::Status& s) {
  if (s.ok()) {
    g_last_error.clear();
    return RS_OK;
  }
  g_last_error = std::string(s.message());
  return s.raw_code();
}

int Bad(const char* what) { return Report(absl::InvalidArgumentError(what)); }

char* Dup(const std::string& s) {
  char* out = static_cast<char*>(std::malloc(s.size() + 1));
  std::memcpy(out, s.c_str(), s.size() + 1);
  return out;
}

}  // namespace

extern "C" {

const char* rs_last_error(void) { return g_last_error.c_str(); }
const char* rs_version(void) { return "redsynth-b200 0.1 (sm_100a)"; }

int rs_ctx_create(int K, const int* cuda_ordinals, size_t max_bytes, rs_ctx** out) {
  if (!out) return Bad("out is null");
  rs::Context* c = nullptr;
  const absl::Status s = rs::CreateContext(K, cuda_ordinals, max_bytes, &c);
  if (s.ok()) *out = new rs_ctx{c};
  return Report(s);
}

int rs_ctx_create_rank(int K, const int* slot_rank, int world_size, int rank, int cuda_ordinal,
                       size_t max_bytes, rs_ctx** out) {
  if (!out) return Bad("out is null");
  rs::Context* c = nullptr;
  const absl::Status s =
      rs::CreateRankContext(K, slot_rank, world_size, rank, cuda_ordinal, max_bytes, &c);
  if (s.ok()) *out = new rs_ctx{c};
  return Report(s);
}

int rs_ctx_create_emulated(int K, const int* slot_rank, int world_size, int cuda_ordinal, size_t max_bytes,
                           rs_ctx** out) {
  if (!out || !slot_rank) return Bad("null argument");
  rs::Context* c = nullptr;
  const absl::Status s = rs::CreateEmulatedContext(K, slot_rank, world_size, cuda_ordinal, max_bytes, &c);
  if (s.ok()) *out = new rs_ctx{c};
  return Report(s);
}

int rs_ctx_create_virtual(int K, const int* slot_rank, int world_size, rs_ctx** out) {
  if (!out || !slot_rank) return Bad("null argument");
  rs::Context* c = nullptr;
  const absl::Status s = rs::CreateVirtualContext(K, slot_rank, world_size, &c);
  if (s.ok()) *out = new rs_ctx{c};
  return Report(s);
}

int rs_ctx_ipc_handle(rs_ctx* ctx, void* out) {
  if (!ctx || !out) return Bad("null argument");
  return Report(rs::IpcHandle(ctx->impl, out));
}

int rs_ctx_open_peers(rs_ctx* ctx, const void* handles) {
  if (!ctx || !handles) return Bad("null argument");
  return Report(rs::OpenPeers(ctx->impl, handles));
}

int rs_ctx_destroy(rs_ctx* ctx) {
  if (!ctx) return RS_OK;
  const absl::Status s = rs::DestroyContext(ctx->impl);
  delete ctx;
  return Report(s);
}

int rs_ctx_buffer(rs_ctx* ctx, int slot, void** device_ptr) {
  if (!ctx || !device_ptr) return Bad("null argument");
  rs::Context* c = ctx->impl;
  if (slot < 0 || slot >= c->K) return Bad("slot out of range");
  const int r = c->slot_rank[slot];
  if (!c->ranks[r].driven) return Bad("slot is not hosted by this process");
  *device_ptr = c->SlotPtr(r, slot);
  return RS_OK;
}

static int CopySlot(rs_ctx* ctx, int slot, void* host, size_t bytes, void* stream, bool up) {
  if (!ctx || !host) return Bad("null argument");
  rs::Context* c = ctx->impl;
  if (slot < 0 || slot >= c->K) return Bad("slot out of range");
  const int r = c->slot_rank[slot];
  if (!c->ranks[r].driven) return Bad("slot is not hosted by this process");
  if (bytes > c->max_bytes) return Bad("copy larger than max_bytes");
  absl::Status s = rs::CudaStatus(cudaSetDevice(c->ranks[r].ordinal), "cudaSetDevice");
  if (!s.ok()) return Report(s);
  cudaStream_t st = stream ? static_cast<cudaStream_t>(stream) : c->ranks[r].stream;
  void* dev = c->SlotPtr(r, slot);
  return Report(rs::CudaStatus(up ? cudaMemcpyAsync(dev, host, bytes, cudaMemcpyHostToDevice, st)
                                  : cudaMemcpyAsync(host, dev, bytes, cudaMemcpyDeviceToHost, st),
                               up ? "upload" : "download"));
}

int rs_ctx_upload(rs_ctx* ctx, int slot, const void* host, size_t bytes, void* stream) {
  return CopySlot(ctx, slot, const_cast<void*>(host), bytes, stream, true);
}

int rs_ctx_download(rs_ctx* ctx, int slot, void* host, size_t bytes, void* stream) {
  return CopySlot(ctx, slot, host, bytes, stream, false);
}

int rs_ctx_local_ranks(rs_ctx* ctx, int* count, int* ordinals) {
  if (!ctx || !count) return Bad("null argument");
  const std::vector<int> driven = ctx->impl->DrivenRanks();
  *count = static_cast<int>(driven.size());
  if (ordinals)
    for (size_t i = 0; i < driven.size(); ++i) ordinals[i] = ctx->impl->ranks[driven[i]].ordinal;
  return RS_OK;
}

int rs_ctx_synchronize(rs_ctx* ctx) {
  if (!ctx) return Bad("null argument");
  return Report(rs::Synchronize(ctx->impl));
}

int rs_plan_compile(rs_ctx* ctx, int num_steps, const int32_t* step_op,
                    const int32_t* step_group_ptr, const int32_t* group_member_ptr,
                    const int32_t* members, size_t elems_per_device, int dtype, rs_plan** out) {
  if (!ctx || !out) return Bad("null argument");
  rs::Plan* p = nullptr;
  const absl::Status s = rs::CompilePlan(ctx->impl, num_steps, step_op, step_group_ptr,
                                         group_member_ptr, members, elems_per_device, dtype, &p);
  if (s.ok()) *out = new rs_plan{p};
  return Report(s);
}

int rs_plan_run(rs_plan* plan, void* const* device_bufs, void* const* streams) {
  if (!plan) return Bad("null plan");
  return Report(rs::RunPlan(plan->impl, device_bufs, nullptr, streams));
}

int rs_plan_run_host(rs_plan* plan, void* const* host_bufs, void* const* streams) {
  if (!plan || !host_bufs) return Bad("null argument");
  return Report(rs::RunPlan(plan->impl, nullptr, host_bufs, streams));
}

int rs_plan_time(rs_plan* plan, int warmup, int iters, double* us) {
  if (!plan || !us || iters < 1 || warmup < 0) return Bad("bad argument");
  rs::Plan* p = plan->impl;
  const std::vector<int> driven = p->ctx->DrivenRanks();
  for (int i = 0; i < warmup; ++i) {
    absl::Status s = rs::RunPlan(p, nullptr, nullptr, nullptr);
    if (!s.ok()) return Report(s);
  }
  std::vector<cudaEvent_t> e0(driven.size()), e1(driven.size());
  for (size_t i = 0; i < driven.size(); ++i) {
    const rs::Rank& rk = p->ctx->ranks[driven[i]];
    cudaSetDevice(rk.ordinal);
    cudaEventCreate(&e0[i]);
    cudaEventCreate(&e1[i]);
    cudaEventRecord(e0[i], rk.stream);
  }
  for (int i = 0; i < iters; ++i) {
    absl::Status s = rs::RunPlan(p, nullptr, nullptr, nullptr);
    if (!s.ok()) return Report(s);
  }
  float worst = 0.f;
  for (size_t i = 0; i < driven.size(); ++i) {
    const rs::Rank& rk = p->ctx->ranks[driven[i]];
    cudaSetDevice(rk.ordinal);
    cudaEventRecord(e1[i], rk.stream);
    cudaEventSynchronize(e1[i]);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0[i], e1[i]);
    worst = std::max(worst, ms);
    cudaEventDestroy(e0[i]);
    cudaEventDestroy(e1[i]);
  }
  *us = 1e3 * worst / iters;
  return Report(rs::Synchronize(p->ctx));
}

int rs_plan_launch_count(rs_plan* plan, int* launches) {
  if (!plan || !launches) return Bad("null argument");
  const rs::Context* c = plan->impl->ctx;
  *launches = plan->impl->num_phases() * (c->emulated ? 1 : static_cast<int>(c->DrivenRanks().size()));
  return RS_OK;
}

int rs_plan_step_bytes(rs_plan* plan, int step, double* link_bytes, double* hbm_bytes) {
  if (!plan) return Bad("null plan");
  const rs::Plan* p = plan->impl;
  if (step < 0 || step >= p->num_steps) return Bad("step out of range");
  double link = 0, hbm = 0;
  for (int ph = 0; ph < p->num_phases(); ++ph) {
    if (p->phase_step[ph] != step) continue;
    double l = 0, h = 0;
    for (const rs::RankStep& r : p->phases[ph]) {
      l = std::max(l, std::max(r.tx_bytes, r.rx_bytes));
      h = std::max(h, r.hbm_bytes);
    }
    link += l;
    hbm += h;
  }
  if (link_bytes) *link_bytes = link;
  if (hbm_bytes) *hbm_bytes = hbm;
  return RS_OK;
}

int rs_plan_predict_us(rs_plan* plan, double launch_us, double link_gbs, double hbm_gbs, double* us) {
  if (!plan || !us) return Bad("null argument");
  if (!(link_gbs > 0) || !(hbm_gbs > 0) || launch_us < 0) return Bad("bandwidths must be positive");
  const rs::Plan* p = plan->impl;
  double total = 0;
  for (const std::vector<rs::RankStep>& phase : p->phases) {
    double link = 0, hbm = 0;
    for (const rs::RankStep& r : phase) {
      link = std::max(link, std::max(r.tx_bytes, r.rx_bytes));
      hbm = std::max(hbm, r.hbm_bytes);
    }
    total += launch_us + link / (link_gbs * 1e3) + hbm / (hbm_gbs * 1e3);
  }
  *us = total;
  return RS_OK;
}

int rs_ctx_set_option(rs_ctx* ctx, const char* key, long long value) {
  if (!ctx || !key) return Bad("null argument");
  const std::string k(key);
  if (k == "push_min_bytes") {
    ctx->impl->push_min_bytes = value < 0 ? ~0ull : static_cast<uint64_t>(value);
  } else if (k == "barrier_timeout_ms") {
    if (value <= 0) return Bad("barrier_timeout_ms must be positive");
    ctx->impl->timeout_ns = static_cast<uint64_t>(value) * 1000000ull;
  } else if (k == "nvls") {
    if (value && !ctx->impl->use_vmm && !ctx->impl->is_virtual) {
      return Bad("NVLS needs a multicast-capable heap: create the context with RS_NVLS=1");
    }
    ctx->impl->nvls = value != 0;
  } else if (k == "nvls_min_group") {
    if (value < 2) return Bad("nvls_min_group must be >= 2");
    ctx->impl->nvls_min_group = static_cast<int>(value);
  } else if (k == "nvls_min_bytes") {
    ctx->impl->nvls_min_bytes = value < 0 ? ~0ull : static_cast<uint64_t>(value);
    ctx->impl->nvls_min_bytes_n8 = ctx->impl->nvls_min_bytes;
  } else if (k == "ll_max_bytes") {
    ctx->impl->ll_max_bytes = value < 0 ? 0 : static_cast<uint64_t>(value);
  } else if (k == "ll_total_bytes") {
    ctx->impl->ll_total_bytes = value < 0 ? 0 : static_cast<uint64_t>(value);
  } else if (k == "push_wave_bytes") {
    ctx->impl->push_wave_bytes = value <= 0 ? 0 : (static_cast<uint64_t>(value) & ~15ull);
  } else if (k == "reduce_mode") {
    if (value < rs::kReduceAuto || value > rs::kReducePushRootPulled) {
      return Bad("reduce_mode must be -1 (auto), 0 (pull), 1 (push), 2 (nvls), 3 (nvls root) or 4 (push, root pulled)");
    }
    ctx->impl->reduce_mode = static_cast<int>(value);
  } else if (k == "nvls_bcast") {
    ctx->impl->nvls_bcast = value != 0;
  } else if (k == "reduce_push_min_bytes") {
    ctx->impl->reduce_push_min_bytes = value < 0 ? ~0ull : static_cast<uint64_t>(value);
  } else if (k == "wave_lag") {
    if (value < 0 || value > 64) return Bad("wave_lag must be in [0, 64]");
    ctx->impl->wave_lag = static_cast<int>(value);
  } else if (k == "reduce_wave_bytes") {
    ctx->impl->reduce_wave_bytes = value <= 0 ? 0 : (static_cast<uint64_t>(value) & ~15ull);
  } else {
    return Bad("unknown option (push_min_bytes | barrier_timeout_ms | nvls | nvls_min_group | nvls_min_bytes | ll_max_bytes | ll_total_bytes | nvls_bcast | reduce_mode | reduce_push_min_bytes | reduce_wave_bytes | push_wave_bytes | wave_lag)");
  }
  return RS_OK;
}

int rs_ctx_set_exchange(rs_ctx* ctx, rs_exchange_fn fn, void* user) {
  if (!ctx) return Bad("null argument");
  ctx->impl->exchange = fn;
  ctx->impl->exchange_user = user;
  return RS_OK;
}

int rs_ctx_nvls(rs_ctx* ctx, int* enabled) {
  if (!ctx || !enabled) return Bad("null argument");
  *enabled = ctx->impl->nvls ? 1 : 0;
  return RS_OK;
}

int rs_plan_set_launch(rs_plan* plan, int max_ctas, int threads) {
  if (!plan) return Bad("null plan");
  if (threads != 0 && (threads < 32 || threads > 512 || threads % 32 != 0)) {
    return Bad("threads must be a multiple of 32 in [32, 512]");
  }
  if (threads != 0) plan->impl->threads = threads;
  plan->impl->max_ctas = max_ctas < 0 ? 0 : max_ctas;
  plan->impl->ctas_per_sm = 0;
  return RS_OK;
}

int rs_plan_set_option(rs_plan* plan, const char* key, long long value) {
  if (!plan || !key) return Bad("null argument");
  const std::string k(key);
  if (k == "unroll") {
    if (value != 4 && value != 8) return Bad("unroll must be 4 or 8");
    plan->impl->unroll = static_cast<int>(value);
  } else if (k == "threads") {
    return rs_plan_set_launch(plan, plan->impl->max_ctas, static_cast<int>(value));
  } else if (k == "max_ctas") {
    plan->impl->max_ctas = value < 0 ? 0 : static_cast<int>(value);
  } else if (k == "wide_loads") {
    plan->impl->wide_loads = value != 0;
  } else if (k == "dynamic_pieces") {
    plan->impl->dynamic_pieces = value != 0;
  } else if (k == "pdl") {
    plan->impl->pdl = value != 0;
  } else if (k == "local_wide") {
    plan->impl->local_wide = value != 0;
  } else if (k == "remote256") {
    plan->impl->remote256 = value != 0;
  } else if (k == "vec256") {
    plan->impl->vec256 = static_cast<int>(value);
  } else if (k == "push_prefetch") {
    plan->impl->push_prefetch = value != 0;
  } else if (k == "piece_queue") {
    if (value < -1 || value > 2) return Bad("piece_queue must be -1 (auto), 0, 1 or 2");
    plan->impl->piece_queue = static_cast<int>(value);
  } else {
    return Bad("unknown option (unroll | threads | max_ctas | wide_loads | dynamic_pieces | pdl | local_wide | vec256 | remote256 | piece_queue | push_prefetch)");
  }
  plan->impl->ctas_per_sm = 0;
  return RS_OK;
}

int rs_plan_describe_json(rs_plan* plan, char** out_json) {
  if (!plan || !out_json) return Bad("null argument");
  *out_json = Dup(rs::DescribePlan(*plan->impl));
  return RS_OK;
}

int rs_plan_destroy(rs_plan* plan) {
  if (!plan) return RS_OK;
  delete plan->impl;
  delete plan;
  return RS_OK;
}

// ---- planner ------------------------------------------------------------

void rs_free(char* p) { std::free(p); }

int rs_synthesize_json(const char* system_json, const int* axes, int n_axes, const int* reduce,
                       int n_reduce, int size_limit, long long payload_bytes, int algo,
                       char** out_json) {
  if (!system_json || !axes || !reduce || !out_json) return Bad("null argument");
  absl::StatusOr<redsynth::SystemModel> system = redsynth::ParseSystem(system_json);
  if (!system.ok()) return Report(system.status());
  redsynth::ParallelismSpec spec;
  spec.axes.assign(axes, axes + n_axes);
  spec.reduction_axes.assign(reduce, reduce + n_reduce);
  absl::StatusOr<std::vector<redsynth::ParallelismMatrix>> matrices =
      redsynth::EnumerateMatrices(*system, spec);
  if (!matrices.ok()) return Report(matrices.status());
  nlohmann::ordered_json doc;
  doc["device_count"] = system->device_count();
  doc["matrices"] = nlohmann::ordered_json::array();
  for (const redsynth::ParallelismMatrix& m : *matrices) {
    nlohmann::ordered_json sec;
    std::vector<std::vector<int>> factors;
    for (int a = 0; a < m.num_axes(); ++a) factors.push_back(m.AxisRow(a));
    sec["factors"] = factors;
    sec["partition"] = redsynth::ReductionGroupPartition(m, spec.reduction_axes, *system);
    redsynth::SynthesisConfig cfg;
    cfg.size_limit = size_limit;
    absl::StatusOr<redsynth::SynthesisResult> res =
        redsynth::Synthesize(m, spec.reduction_axes, *system, cfg);
    if (!res.ok()) return Report(res.status());
    std::vector<std::string> labels;
    for (const auto& l : res->hierarchy.levels) labels.push_back(l.label);
    sec["hierarchy"] = labels;
    sec["programs"] = nlohmann::ordered_json::array();
    redsynth::CostModelConfig cost;
    cost.algo = algo == 1 ? redsynth::CollectiveAlgo::kTree : redsynth::CollectiveAlgo::kRing;
    cost.payload_bytes = payload_bytes;
    for (const redsynth::SynthesizedProgram& p : res->programs) {
      nlohmann::ordered_json e;
      e["text"] = redsynth::PrettyPrint(p.program, res->hierarchy);
      absl::StatusOr<redsynth::CostReport> sim = redsynth::Simulate(p.lowered, *system, cost);
      e["seconds"] = sim.ok() ? sim->total_seconds : -1.0;
      e["steps"] = nlohmann::ordered_json::array();
      for (const redsynth::CollectiveStep& st : p.lowered.steps) {
        e["steps"].push_back({{"op", static_cast<int>(st.op)}, {"groups", st.groups}});
      }
      sec["programs"].push_back(std::move(e));
    }
    doc["matrices"].push_back(std::move(sec));
  }
  *out_json = Dup(doc.dump());
  return RS_OK;
}

int rs_report(const char* system_path, const int* axes, int n_axes, const int* reduce,
              int n_reduce, int size_limit, long long payload_bytes, int algo, int csv,
              char** out) {
  if (!system_path || !axes || !reduce || !out) return Bad("null argument");
  redsynth::RunRequest req;
  req.system_path = system_path;
  req.axes.assign(axes, axes + n_axes);
  req.reduction_axes.assign(reduce, reduce + n_reduce);
  req.algo = algo == 1 ? redsynth::CollectiveAlgo::kTree : redsynth::CollectiveAlgo::kRing;
  req.payload_bytes = payload_bytes;
  req.size_limit = size_limit;
  absl::StatusOr<redsynth::Report> rep = redsynth::RunPipeline(req);
  if (!rep.ok()) return Report(rep.status());
  *out = Dup(csv ? redsynth::ReportToCsv(*rep) : redsynth::ReportToJson(*rep));
  return RS_OK;
}

int rs_run_lowered(int num_steps, const int32_t* step_op, const int32_t* step_group_ptr,
                   const int32_t* group_member_ptr, const int32_t* members, int k,
                   unsigned char* state, int* fail_step, int* fail_violation) {
  redsynth::LoweredProgram lowered;
  for (int s = 0; s < num_steps; ++s) {
    redsynth::CollectiveStep step;
    step.op = static_cast<redsynth::Collective>(step_op[s]);
    for (int g = step_group_ptr[s]; g < step_group_ptr[s + 1]; ++g)
      step.groups.emplace_back(members + group_member_ptr[g], members + group_member_ptr[g + 1]);
    lowered.steps.push_back(std::move(step));
  }
  redsynth::StepFailure failure;
  absl::StatusOr<redsynth::StateContext> ctx = redsynth::RunLowered(lowered, k, &failure);
  if (!ctx.ok()) {
    if (fail_step) *fail_step = failure.step;
    if (fail_violation) *fail_violation = static_cast<int>(failure.violation);
    return Report(ctx.status());
  }
  if (state) {
    for (int d = 0; d < k; ++d)
      for (int r = 0; r < k; ++r)
        for (int c = 0; c < k; ++c)
          state[(static_cast<size_t>(d) * k + r) * k + c] = ctx->state(d).bit(r, c) ? 1 : 0;
  }
  return RS_OK;
}

}  // extern "C"
