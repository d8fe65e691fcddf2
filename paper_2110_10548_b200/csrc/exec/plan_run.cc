// Plan execution: launch records, the per-run launch path and the JSON
// description of a compiled plan (compilation: plan.cc).
#include <algorithm>
#include <cstdlib>

#include "absl/strings/str_format.h"
#include "exec_internal.h"
#include "nlohmann/json.hpp"

namespace rs {

Plan::~Plan() {
  if (!ctx) return;
  for (size_t r = 0; r < d_tasks.size(); ++r) {
    if (!ctx->ranks[r].driven) continue;
    cudaSetDevice(ctx->ranks[r].ordinal);
    if (d_tasks[r]) cudaFree(d_tasks[r]);
    if (d_ptrs[r]) cudaFree(d_ptrs[r]);
  }
}

// Launch records of every (phase, driven rank), built once per launch shape
// (the per-run host path is then one launch per record).
void BuildLaunches(Plan* plan) {
  Context* ctx = plan->ctx;
#ifdef RS_PROFILING_AIDS
  const char* solo_env = std::getenv("RS_SOLO_PROFILE");
  const bool solo = solo_env && std::atoi(solo_env) != 0;
#endif
  const int P = plan->num_phases();
  const int R = ctx->world;
  plan->launch_args.assign(static_cast<size_t>(P) * R, StepArgs{});
  plan->launch_grid.assign(static_cast<size_t>(P) * R, 1);
  for (int ph = 0; ph < P; ++ph) {
    for (int r : ctx->DrivenRanks()) {
      const Rank& rank = ctx->ranks[r];
      const RankStep& rsx = plan->phases[ph][r];
      StepArgs& a = plan->launch_args[static_cast<size_t>(ph) * R + r];
      a.tasks = plan->d_tasks[r] ? plan->d_tasks[r] + plan->task_offset[r][ph] : nullptr;
      a.ptrs = plan->d_ptrs[r] ? plan->d_ptrs[r] + plan->ptr_offset[r][ph] : nullptr;
      a.ntasks = static_cast<uint32_t>(rsx.tasks.size());
      a.npieces = rsx.npieces;
      a.piece_bytes = rsx.piece_bytes;
      a.dtype = plan->dtype;
      a.arrive_counter = reinterpret_cast<unsigned int*>(rank.heap + kCounterOffset);
      a.error_flag = reinterpret_cast<int*>(rank.heap + kErrorOffset);
      a.inbox = reinterpret_cast<const uint64_t*>(rank.heap + kInboxOffset);
      a.timeout_ns = ctx->timeout_ns;
      a.ll_parity_stride = ctx->LLRegionBytes();
      a.flag_chunk = static_cast<uint32_t>(ctx->flag_chunk);
      a.recv_piece = rsx.recv_piece;
      if (ctx->world > 1) {
        for (int q = 0; q < ctx->world; ++q) {
          if (q == r) continue;
          a.signal_ptrs[a.nsignal++] = reinterpret_cast<uint64_t*>(rank.view[q] + kInboxOffset) + r;
        }
        for (uint8_t q : rsx.wait) a.wait_ranks[a.nwait++] = q;
        if (ph == P - 1) {
          for (int q = 0; q < ctx->world; ++q)
            if (plan->final_wait_bits[r] & (1u << q)) a.final_ranks[a.nfinal++] = static_cast<uint8_t>(q);
        }
      }
#ifdef RS_PROFILING_AIDS
      if (solo) {
        // Profiling builds only (make profiling -> libredsynth_b200_prof.so):
        // with RS_SOLO_PROFILE=1 no cross-GPU waits, so ncu can replay one
        // GPU's pull/push kernel alone and count its NVLink bytes (results
        // are garbage). The release library has no such switch.
        a.nwait = 0;
        a.nfinal = 0;
        a.solo = 1;
      }
      // Piece timeline (tools/trace_push.py): RS_TRACE_PTR = device address
      // of a buffer on this rank's GPU, >= 3 * npieces + 2 * grid uint64.
      if (const char* tp = std::getenv("RS_TRACE_PTR")) a.trace = reinterpret_cast<uint64_t*>(std::strtoull(tp, nullptr, 10));
#endif
      a.local_only = ctx->world == 1 ? 1u : 0u;
      a.wide_loads = plan->wide_loads ? 1u : 0u;
      a.pdl = plan->pdl ? 1u : 0u;
      a.local_wide = plan->local_wide ? 1u : 0u;
      a.vec256 = static_cast<uint32_t>(plan->vec256);
      a.remote256 = plan->remote256 ? 1u : 0u;
      a.slot_limit = ctx->slot_stride;
      a.signal_done = rsx.signal_done ? 1u : 0u;
      a.wait_lag = static_cast<uint32_t>(plan->phase_lag[ph]);
      a.epoch_base = reinterpret_cast<uint64_t*>(rank.heap + kEpochOffset);
      a.step = static_cast<uint32_t>(ph);
      a.num_steps = static_cast<uint32_t>(P);
      a.piece_counter = reinterpret_cast<unsigned int*>(rank.heap + kPieceCounterOffset);
      for (const Task& t : rsx.tasks) {
        a.has_nvls |= (t.mode == kModeNvlsAllReduce || t.mode == kModeNvlsReduce || t.mode == kModeNvlsBroadcast) ? 1u : 0u;
        a.has_ll |= t.mode == kModeLL ? 1u : 0u;
        a.dynamic |= (plan->dynamic_pieces && (t.mode == kModeFlagSend || t.mode == kModeFlagRecv)) ? 1u : 0u;
      }
      // piece_queue 1: this rank's phase touches only its own HBM (every
      // phase of a one-GPU context, the GPU-local steps of multi-GPU ones);
      // 2: also pull phases. NVLS and one-shot phases keep the static stride
      // (NVLS was not A/B'd with the queue).
      // -1 (auto, default): 1, plus pull phases where that was measured
      // faster (2 and 4 real GPUs; emulated 8 ranks on one GPU: -5 %).
      const bool own_hbm = rsx.remote_peers == 0;
      const bool pull_q = plan->piece_queue >= 2 || (plan->piece_queue < 0 && !ctx->emulated && R <= 4);
      if (a.dynamic == 0 && !a.has_ll && !a.has_nvls && plan->piece_queue != 0 && (own_hbm || pull_q))
        a.dynamic = 2;
      int resident = plan->ctas_per_sm * rank.sm_count;
      if (ctx->emulated) {
        // all ranks share one cooperative launch: split its co-resident CTAs
        const bool ll = plan->phase_ll[ph] != 0;
        resident = std::max(1, EmulatedResidentCtas(plan->dtype, plan->threads, ll) * rank.sm_count / R);
      }
      int cap = plan->max_ctas > 0 ? std::min(plan->max_ctas, resident) : resident;
      if (rsx.max_grid > 0) cap = std::min<int>(cap, static_cast<int>(rsx.max_grid));
      // Pulling from >= 2 peers at once: one CTA per SM keeps fewer loads in
      // flight and measured +6 % at K=4 (637 vs 597 GB/s bus, 256 MiB
      // AllReduce, profiles/r01_tune4_push0.log); from one peer two per SM
      // are better (652 vs 637 at K=2, r01_tune_n2.log).
      if (plan->max_ctas == 0 && !a.has_nvls && !a.has_ll && rsx.remote_peers >= 2) cap = std::min(cap, rank.sm_count);
      if (cap <= 0) cap = std::max(1, rank.sm_count);
      const bool push_queue = a.dynamic == 1;  // ordering required: never static
      if (push_queue && plan->push_prefetch) a.dynamic = 2;
      const int grid = std::max(1, std::min<int>(cap, static_cast<int>(rsx.npieces)));
      plan->launch_grid[static_cast<size_t>(ph) * R + r] = grid;
      // Under two pieces per CTA there is nothing to balance and the queue's
      // first atomic is pure latency (K=4 1 MiB AllReduce 16.6 -> 19.3 us).
      if (a.dynamic == 2 && !push_queue && rsx.npieces < 2u * static_cast<uint32_t>(grid)) a.dynamic = 0;
    }
  }
}

absl::Status RunPlan(Plan* plan, void* const* device_bufs, void* const* host_bufs,
                     void* const* streams) {
  Context* ctx = plan->ctx;
  if (ctx->is_virtual) return absl::FailedPreconditionError("virtual (planning-only) context cannot run");
  const std::vector<int> driven = ctx->DrivenRanks();
  auto stream_of = [&](size_t i) {
    return streams ? static_cast<cudaStream_t>(streams[i]) : ctx->ranks[driven[i]].stream;
  };
  auto copy_all = [&](bool in) -> absl::Status {
    for (size_t i = 0; i < driven.size(); ++i) {
      const int r = driven[i];
      absl::Status s = CudaStatus(cudaSetDevice(ctx->ranks[r].ordinal), "cudaSetDevice");
      if (!s.ok()) return s;
      for (int d = 0; d < ctx->K; ++d) {
        if (ctx->slot_rank[d] != r) continue;
        void* user = device_bufs ? device_bufs[d] : host_bufs[d];
        if (!user) return absl::InvalidArgumentError(absl::StrFormat("buffer of slot %d is null", d));
        void* slot = ctx->SlotPtr(r, d);
        const cudaMemcpyKind kind = device_bufs ? cudaMemcpyDeviceToDevice
                                    : in        ? cudaMemcpyHostToDevice
                                                : cudaMemcpyDeviceToHost;
        s = CudaStatus(cudaMemcpyAsync(in ? slot : user, in ? user : slot, plan->bytes, kind, stream_of(i)),
                       in ? "copy-in" : "copy-out");
        if (!s.ok()) return s;
      }
    }
    return absl::OkStatus();
  };
  if (device_bufs || host_bufs) {
    absl::Status s = copy_all(true);
    if (!s.ok()) return s;
  }
  const int P = plan->num_phases();
  if (plan->ctas_per_sm == 0 && !driven.empty()) {
    absl::Status st = CudaStatus(cudaSetDevice(ctx->ranks[driven[0]].ordinal), "cudaSetDevice");
    if (!st.ok()) return st;
    plan->ctas_per_sm = MaxResidentCtas(plan->dtype, plan->threads, plan->unroll);
    BuildLaunches(plan);
  }
  const int R = ctx->world;
  if (driven.size() == 1) {
    absl::Status st = CudaStatus(cudaSetDevice(ctx->ranks[driven[0]].ordinal), "cudaSetDevice");
    if (!st.ok()) return st;
  }
  if (ctx->emulated) {
    // one cooperative launch per phase covering every rank (stream of rank 0)
    for (int ph = 0; ph < P; ++ph) {
      EmulatedArgs e{};
      e.nranks = static_cast<uint32_t>(R);
      bool ll = false;
      for (int r = 0; r < R; ++r) {
        const size_t k = static_cast<size_t>(ph) * R + r;
        e.args[r] = plan->launch_args[k];
        e.prefix[r + 1] = e.prefix[r] + static_cast<uint32_t>(plan->launch_grid[k]);
        ll |= e.args[r].has_ll != 0;
      }
      absl::Status st = CudaStatus(LaunchEmulated(e, ll, plan->threads, stream_of(0)), "emulated step launch");
      if (!st.ok()) return st;
    }
    if (device_bufs || host_bufs) return copy_all(false);
    return absl::OkStatus();
  }
  for (int ph = 0; ph < P; ++ph) {
    for (size_t i = 0; i < driven.size(); ++i) {
      const int r = driven[i];
      if (driven.size() > 1) {
        absl::Status st = CudaStatus(cudaSetDevice(ctx->ranks[r].ordinal), "cudaSetDevice");
        if (!st.ok()) return st;
      }
      const size_t k = static_cast<size_t>(ph) * R + r;
      absl::Status st = CudaStatus(
          LaunchStep(plan->launch_args[k], plan->launch_grid[k], plan->threads, plan->unroll, stream_of(i)),
          "step kernel launch");
      if (!st.ok()) return st;
    }
  }
  if (device_bufs || host_bufs) return copy_all(false);
  return absl::OkStatus();
}

std::string DescribePlan(const Plan& plan) {
  nlohmann::ordered_json doc;
  doc["num_steps"] = plan.num_steps;
  doc["num_phases"] = plan.num_phases();
  doc["phase_step"] = plan.phase_step;
  doc["phase_ll"] = plan.phase_ll;
  doc["phase_lag"] = plan.phase_lag;
  doc["bytes"] = plan.bytes;
  doc["world"] = plan.ctx->world;
  doc["slot_rank"] = plan.ctx->slot_rank;
  doc["scratch_regions"] = plan.ctx->scratch_regions;
  nlohmann::ordered_json phases = nlohmann::ordered_json::array();
  const size_t R = static_cast<size_t>(plan.ctx->world);
  for (size_t ph = 0; ph < plan.phases.size(); ++ph) {
    const std::vector<RankStep>& per_rank = plan.phases[ph];
    nlohmann::ordered_json ranks = nlohmann::ordered_json::array();
    for (size_t ri = 0; ri < per_rank.size(); ++ri) {
      const RankStep& r = per_rank[ri];
      nlohmann::ordered_json tasks = nlohmann::ordered_json::array();
      for (const Task& t : r.tasks) {
        std::vector<int> src, dst, src_region, dst_region, sends;
        for (int i = 0; i < t.nsrc + t.ndst; ++i) {
          const Ref& ref = r.ptr_refs[t.ptr_begin + i];
          if (i >= t.nsrc && ref.region == kLLRegion) {
            sends.push_back(ref.ll_recv);  // packets of the local source to that rank
            continue;
          }
          (i < t.nsrc ? src : dst).push_back(ref.slot);
          (i < t.nsrc ? src_region : dst_region).push_back(ref.region);
        }
        if (t.mode == kModeLL) {
          tasks.push_back({{"lo", t.lo}, {"hi", t.hi}, {"vec", t.vec}, {"mode", t.mode},
                           {"piece_begin", t.piece_begin}, {"src", src}, {"dst", dst}, {"src_region", src_region},
                           {"dst_region", dst_region}, {"sends", sends}});
          continue;
        }
        if (t.mode == kModeNvlsBroadcast) {
          const McGroup* mc = plan.ctx->mc_index[r.ptr_refs[t.ptr_begin + 1].slot];
          std::vector<int> mdst(mc->slots.begin() + 1, mc->slots.end());
          tasks.push_back({{"lo", t.lo}, {"hi", t.hi}, {"vec", t.vec}, {"mode", t.mode},
                           {"piece_begin", t.piece_begin}, {"src", std::vector<int>{mc->slots[0]}}, {"dst", mdst},
                           {"src_region", std::vector<int>{-1}}, {"dst_region", std::vector<int>(mdst.size(), -1)}});
          continue;
        }
        if (t.mode == kModeNvlsAllReduce || t.mode == kModeNvlsReduce) {
          const McGroup* mc = plan.ctx->mc_index[r.ptr_refs[t.ptr_begin].slot];
          std::vector<int> mdst = mc->slots;
          if (t.mode == kModeNvlsReduce) {
            mdst.clear();
            for (int i = 0; i < t.ndst; ++i) mdst.push_back(r.ptr_refs[t.ptr_begin + 1 + i].slot);
          }
          tasks.push_back({{"lo", t.lo}, {"hi", t.hi}, {"vec", t.vec}, {"mode", t.mode},
                           {"piece_begin", t.piece_begin}, {"src", mc->slots}, {"dst", mdst},
                           {"src_region", std::vector<int>(mc->slots.size(), -1)},
                           {"dst_region", std::vector<int>(mdst.size(), -1)}});
          continue;
        }
        tasks.push_back({{"lo", t.lo}, {"hi", t.hi}, {"vec", t.vec}, {"mode", t.mode}, {"piece_begin", t.piece_begin},
                         {"src", src}, {"dst", dst}, {"src_region", src_region},
                         {"dst_region", dst_region}});
      }
      std::vector<int> wait(r.wait.begin(), r.wait.end());
      ranks.push_back({{"wait", wait}, {"signal", r.signal_done}, {"npieces", r.npieces}, {"tx", r.tx_bytes}, {"rx", r.rx_bytes},
                       {"hbm", r.hbm_bytes}, {"tasks", tasks}});
      // After the first run on a driven rank: the launch shape and the piece
      // schedule (0 static grid stride, 1 push queue, 2 prefetched queue).
      const size_t k = ph * R + ri;
      if (k < plan.launch_args.size() && plan.launch_args[k].piece_counter != nullptr) {
        ranks.back()["grid"] = plan.launch_grid[k];
        ranks.back()["queue"] = plan.launch_args[k].dynamic;
      }
    }
    phases.push_back({{"ranks", ranks}});
  }
  doc["steps"] = std::move(phases);  // launch phases: one per program step
  std::vector<std::vector<int>> final_wait;
  for (uint8_t bits : plan.final_wait_bits) {
    std::vector<int> w;
    for (int q = 0; q < RS_MAX_RANKS; ++q)
      if (bits & (1u << q)) w.push_back(q);
    final_wait.push_back(w);
  }
  doc["final_wait"] = final_wait;
  return doc.dump();
}

}  // namespace rs
