// Plan compiler: LoweredProgram (CSR) -> per-(step, rank) task lists.
//
// 1. Replays the reference semantics step by step (redsynth::
//    ApplyCollectiveInPlace, semantics.cc:259-310, folded as RunLowered does,
//    dsl.cc:142-164) to learn which rows every slot holds before each step and
//    to refuse invalid programs with the reference's step/violation.
// 2. Turns every group of every step into owner tasks (see step_kernel.cu for
//    the per-collective data movement) over row ranges; row r of a slot buffer
//    is elements [floor(rN/K), floor((r+1)N/K)).
// 3. Tracks a content id per (slot, row) so copies whose destination already
//    holds bit-identical data (same id) are skipped — the result is the same
//    bits the oracle's unconditional overwrite produces.
// 4. Computes each rank's entry-barrier set (ranks whose buffers it touches
//    and their previous-step writers) and the tail barrier of the run.
#include <algorithm>
#include <map>
#include <memory>
#include <numeric>
#include <set>
#include <tuple>

#include "absl/strings/str_format.h"
#include "exec_internal.h"
#include "nlohmann/json.hpp"
#include "redsynth/dsl.h"
#include "redsynth/semantics.h"

namespace rs {
namespace {

struct Range {
  uint64_t lo, hi;
};

struct ProtoTask {
  int owner;
  Range range;
  std::vector<int> src;  // slots, summation order
  std::vector<int> dst;  // slots
};

class RowGeometry {
 public:
  RowGeometry(size_t elems, int K, size_t es) : elems_(elems), K_(K), es_(es) {}
  uint64_t Lo(int r) const {
    return static_cast<uint64_t>((static_cast<unsigned __int128>(r) * elems_) / K_) * es_;
  }
  // Maximal runs of consecutive rows -> byte ranges (empty rows dropped).
  std::vector<Range> Ranges(const std::vector<int>& rows) const {
    std::vector<Range> out;
    for (size_t i = 0; i < rows.size();) {
      size_t j = i + 1;
      while (j < rows.size() && rows[j] == rows[j - 1] + 1) ++j;
      Range rg{Lo(rows[i]), Lo(rows[j - 1] + 1)};
      if (rg.hi > rg.lo) out.push_back(rg);
      i = j;
    }
    return out;
  }

 private:
  size_t elems_;
  int K_;
  size_t es_;
};

// Splits the concatenation of `ranges` into k consecutive parts of nearly
// equal size whose cut points sit on 16-byte buffer offsets (or on range
// starts), so owners' vector work stays aligned.
std::vector<std::vector<Range>> SplitEven(const std::vector<Range>& ranges, int k) {
  std::vector<std::vector<Range>> parts(k);
  if (ranges.empty() || k <= 0) return parts;
  uint64_t total = 0;
  for (const Range& r : ranges) total += r.hi - r.lo;
  // Map concatenated coordinate -> aligned concatenated coordinate.
  auto align = [&](uint64_t c) {
    uint64_t base = 0;
    for (const Range& r : ranges) {
      const uint64_t len = r.hi - r.lo;
      if (c < base + len || (&r == &ranges.back())) {
        const uint64_t b = std::min(r.lo + (c - base), r.hi);
        uint64_t a = b & ~uint64_t{15};
        if (a < r.lo) a = r.lo;
        return base + (a - r.lo);
      }
      base += len;
    }
    return total;
  };
  std::vector<uint64_t> cut(k + 1);
  cut[0] = 0;
  cut[k] = total;
  for (int j = 1; j < k; ++j) {
    cut[j] = align(static_cast<uint64_t>((static_cast<unsigned __int128>(total) * j) / k));
    cut[j] = std::max(cut[j], cut[j - 1]);
  }
  for (int j = 0; j < k; ++j) {
    uint64_t base = 0;
    for (const Range& r : ranges) {
      const uint64_t len = r.hi - r.lo;
      const uint64_t a = std::max(cut[j], base), b = std::min(cut[j + 1], base + len);
      if (a < b) parts[j].push_back(Range{r.lo + (a - base), r.lo + (b - base)});
      base += len;
    }
  }
  return parts;
}

std::vector<int> HeldRows(const redsynth::StateContext& st, int d) {
  return st.state(d).NonEmptyRows();
}

struct Compiler {
  Context* ctx;
  int K;
  int S;
  size_t es;
  RowGeometry geo;
  std::vector<uint64_t> vid;  // content id of (slot, row)
  uint64_t next_id;

  Compiler(Context* c, int steps, size_t elems, size_t esize)
      : ctx(c), K(c->K), S(steps), es(esize), geo(elems, c->K, esize), vid(static_cast<size_t>(c->K) * c->K) {
    for (size_t i = 0; i < vid.size(); ++i) vid[i] = i + 1;
    next_id = vid.size() + 1;
  }
  uint64_t& Vid(int d, int r) { return vid[static_cast<size_t>(d) * K + r]; }

  void Emit(std::vector<ProtoTask>& out, const std::vector<Range>& ranges,
            const std::vector<int>& owners, const std::vector<int>& src, const std::vector<int>& dst) {
    const std::vector<std::vector<Range>> parts = SplitEven(ranges, static_cast<int>(owners.size()));
    for (size_t j = 0; j < owners.size(); ++j)
      for (const Range& r : parts[j]) out.push_back(ProtoTask{owners[j], r, src, dst});
  }

  // Copies of rows from their holder to every member whose memory differs.
  void EmitCopies(std::vector<ProtoTask>& out, const std::vector<int>& g,
                  const std::vector<std::pair<int, int>>& row_holder) {
    // Key rows by (holder, receivers) so contiguous rows merge into ranges.
    std::map<std::pair<int, std::vector<int>>, std::vector<int>> by_key;
    for (auto [r, h] : row_holder) {
      std::vector<int> recv;
      for (int m : g)
        if (m != h && Vid(m, r) != Vid(h, r)) recv.push_back(m);
      if (!recv.empty()) by_key[{h, recv}].push_back(r);
    }
    for (auto& [key, rows] : by_key) {
      std::sort(rows.begin(), rows.end());
      Emit(out, geo.Ranges(rows), key.second, {key.first}, key.second);
      for (int r : rows)
        for (int m : key.second) Vid(m, r) = Vid(key.first, r);
    }
  }

  void Group(std::vector<ProtoTask>& out, const redsynth::StateContext& pre,
             const std::vector<int>& g, redsynth::Collective op) {
    using redsynth::Collective;
    const int n = static_cast<int>(g.size());
    switch (op) {
      case Collective::kAllReduce: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        Emit(out, geo.Ranges(rows), g, g, g);
        for (int r : rows) {
          const uint64_t id = next_id++;
          for (int m : g) Vid(m, r) = id;
        }
        break;
      }
      case Collective::kReduceScatter: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const int run = n ? static_cast<int>(rows.size()) / n : 0;
        for (int m = 0; m < n && run > 0; ++m) {
          std::vector<int> mine(rows.begin() + m * run, rows.begin() + (m + 1) * run);
          Emit(out, geo.Ranges(mine), {g[m]}, g, {g[m]});
          for (int r : mine) Vid(g[m], r) = next_id++;
        }
        break;
      }
      case Collective::kReduce: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const std::vector<int> owners(g.begin() + 1, g.end());
        Emit(out, geo.Ranges(rows), owners, g, {g[0]});
        for (int r : rows) Vid(g[0], r) = next_id++;
        break;
      }
      case Collective::kAllGather: {
        std::vector<std::pair<int, int>> row_holder;
        for (int r = 0; r < K; ++r)
          for (int m : g)
            if (!pre.state(m).RowEmpty(r)) row_holder.push_back({r, m});
        EmitCopies(out, g, row_holder);
        break;
      }
      case Collective::kBroadcast: {
        std::vector<std::pair<int, int>> row_holder;
        for (int r : HeldRows(pre, g[0])) row_holder.push_back({r, g[0]});
        EmitCopies(out, g, row_holder);
        break;
      }
    }
  }
};

void AddTraffic(std::vector<RankStep>& per_rank, const Context& ctx, const ProtoTask& t) {
  const double b = static_cast<double>(t.range.hi - t.range.lo);
  const int o = ctx.slot_rank[t.owner];
  for (int x : t.src) {
    const int rx = ctx.slot_rank[x];
    per_rank[rx].hbm_bytes += b;
    if (rx != o) {
      per_rank[o].rx_bytes += b;
      per_rank[rx].tx_bytes += b;
    }
  }
  for (int y : t.dst) {
    const int ry = ctx.slot_rank[y];
    per_rank[ry].hbm_bytes += b;
    if (ry != o) {
      per_rank[o].tx_bytes += b;
      per_rank[ry].rx_bytes += b;
    }
  }
}

// Appends `t` to its owner rank's step: vector body + scalar head/tail.
void Lay(RankStep& rs, const ProtoTask& t, uint32_t piece_bytes) {
  auto push = [&](uint64_t lo, uint64_t hi, bool vec) {
    if (hi <= lo) return;
    Task task{};
    task.lo = lo;
    task.hi = hi;
    task.piece_begin = rs.npieces;
    task.ptr_begin = static_cast<uint32_t>(rs.ptr_slots.size());
    task.nsrc = static_cast<uint16_t>(t.src.size());
    task.ndst = static_cast<uint16_t>(t.dst.size());
    task.vec = vec ? 1u : 0u;
    rs.ptr_slots.insert(rs.ptr_slots.end(), t.src.begin(), t.src.end());
    rs.ptr_slots.insert(rs.ptr_slots.end(), t.dst.begin(), t.dst.end());
    rs.npieces += vec ? static_cast<uint32_t>((hi - lo + piece_bytes - 1) / piece_bytes) : 1u;
    rs.tasks.push_back(task);
  };
  const uint64_t a = (t.range.lo + 15) & ~uint64_t{15};
  const uint64_t b = t.range.hi & ~uint64_t{15};
  if (a >= b) {
    // No aligned body: at most 30 bytes, two scalar tasks keep each < 16 B.
    const uint64_t mid = std::min(std::max(a, t.range.lo), t.range.hi);
    push(t.range.lo, mid, false);
    push(mid, t.range.hi, false);
    return;
  }
  push(t.range.lo, a, false);
  push(a, b, true);
  push(b, t.range.hi, false);
}

}  // namespace

Plan::~Plan() {
  if (!ctx) return;
  for (size_t r = 0; r < d_tasks.size(); ++r) {
    if (!ctx->ranks[r].driven) continue;
    cudaSetDevice(ctx->ranks[r].ordinal);
    if (d_tasks[r]) cudaFree(d_tasks[r]);
    if (d_ptrs[r]) cudaFree(d_ptrs[r]);
  }
}

absl::Status CompilePlan(Context* ctx, int num_steps, const int32_t* step_op,
                         const int32_t* step_group_ptr, const int32_t* group_member_ptr,
                         const int32_t* members, size_t elems, int dtype, Plan** out) {
  using redsynth::Collective;
  if (!ctx->peers_open) return absl::FailedPreconditionError("peers not opened (rs_ctx_open_peers)");
  if (num_steps < 0) return absl::InvalidArgumentError("num_steps must be >= 0");
  if (num_steps > 0 && (!step_op || !step_group_ptr || !group_member_ptr || !members)) {
    return absl::InvalidArgumentError("null program array");
  }
  if (dtype != RS_F32 && dtype != RS_BF16 && dtype != RS_I32) {
    return absl::InvalidArgumentError(absl::StrFormat("unknown dtype %d", dtype));
  }
  const size_t es = dtype == RS_BF16 ? 2 : 4;
  if (elems * es > ctx->max_bytes) {
    return absl::InvalidArgumentError(absl::StrFormat(
        "%d bytes per slot exceed the context's max_bytes (%d)", elems * es, ctx->max_bytes));
  }
  // CSR sanity (memory safety), then the program itself.
  redsynth::LoweredProgram lowered;
  for (int s = 0; s < num_steps; ++s) {
    if (step_op[s] < 0 || step_op[s] > 4) {
      return absl::InvalidArgumentError(absl::StrFormat("step %d: unknown collective %d", s, step_op[s]));
    }
    if (step_group_ptr[s + 1] < step_group_ptr[s]) {
      return absl::InvalidArgumentError("step_group_ptr must be non-decreasing");
    }
    redsynth::CollectiveStep step;
    step.op = static_cast<Collective>(step_op[s]);
    for (int g = step_group_ptr[s]; g < step_group_ptr[s + 1]; ++g) {
      if (group_member_ptr[g + 1] < group_member_ptr[g]) {
        return absl::InvalidArgumentError("group_member_ptr must be non-decreasing");
      }
      step.groups.emplace_back(members + group_member_ptr[g], members + group_member_ptr[g + 1]);
    }
    lowered.steps.push_back(std::move(step));
  }

  // 1. Reference semantics, step by step (RunLowered's fold).
  const int K = ctx->K;
  std::vector<redsynth::StateContext> pre;
  redsynth::StateContext st = redsynth::InitialContext(K);
  for (int s = 0; s < num_steps; ++s) {
    const redsynth::CollectiveStep& step = lowered.steps[s];
    if (step.groups.empty()) {
      return absl::InvalidArgumentError(absl::StrFormat("step %d has no device groups", s));
    }
    pre.push_back(st);
    for (const std::vector<int>& g : step.groups) {
      const redsynth::RuleViolation v = redsynth::ApplyCollectiveInPlace(st, g, step.op);
      if (v != redsynth::RuleViolation::kNone) {
        redsynth::StepFailure f;
        f.step = s;
        f.op = step.op;
        f.violation = v;
        f.group = g;
        return absl::FailedPreconditionError(f.Describe());
      }
    }
    std::vector<int> seen(K, 0);
    for (const std::vector<int>& g : step.groups) {
      for (int d : g) {
        if (seen[d]++) {
          return absl::InvalidArgumentError(absl::StrFormat(
              "step %d: device %d appears in two groups (groups of a step must be disjoint)", s, d));
        }
      }
    }
  }

  auto plan = std::make_unique<Plan>();
  plan->ctx = ctx;
  plan->num_steps = num_steps;
  plan->dtype = dtype;
  plan->elems = elems;
  plan->bytes = elems * es;
  const uint32_t piece_bytes = kPieceBytes;

  // 2./3. Tasks per step.
  Compiler comp(ctx, num_steps, elems, es);
  const int R = ctx->world;
  plan->steps.assign(num_steps, std::vector<RankStep>(R));
  // group index of each slot per step (-1 = idle)
  std::vector<std::vector<int>> gidx(num_steps, std::vector<int>(K, -1));
  for (int s = 0; s < num_steps; ++s) {
    std::vector<ProtoTask> tasks;
    const redsynth::CollectiveStep& step = lowered.steps[s];
    for (size_t gi = 0; gi < step.groups.size(); ++gi) {
      for (int d : step.groups[gi]) gidx[s][d] = static_cast<int>(gi);
      comp.Group(tasks, pre[s], step.groups[gi], step.op);
    }
    for (const ProtoTask& t : tasks) {
      AddTraffic(plan->steps[s], *ctx, t);
      Lay(plan->steps[s][ctx->slot_rank[t.owner]], t, piece_bytes);
    }
  }

  // 4. Barrier sets.
  auto group_of = [&](int s, int d) -> std::vector<int> {
    if (s < 0 || gidx[s][d] < 0) return {d};
    return lowered.steps[s].groups[gidx[s][d]];
  };
  plan->final_wait_bits.assign(R, 0);
  for (int s = 0; s < num_steps; ++s) {
    for (int r = 0; r < R; ++r) {
      std::set<int> wait;
      for (int d = 0; d < K; ++d) {
        if (ctx->slot_rank[d] != r) continue;
        for (int q : group_of(s, d))
          for (int p : group_of(s - 1, q)) wait.insert(ctx->slot_rank[p]);
      }
      wait.erase(r);
      plan->steps[s][r].wait.assign(wait.begin(), wait.end());
    }
  }
  if (num_steps > 0) {
    for (int d = 0; d < K; ++d) {
      const int r = ctx->slot_rank[d];
      for (int p : group_of(num_steps - 1, d)) {
        const int q = ctx->slot_rank[p];
        if (q != r) plan->final_wait_bits[r] |= static_cast<uint8_t>(1u << q);
      }
    }
  }

  // Device copies for every rank this process drives.
  plan->d_tasks.assign(R, nullptr);
  plan->d_ptrs.assign(R, nullptr);
  plan->task_offset.assign(R, std::vector<size_t>(num_steps, 0));
  plan->ptr_offset.assign(R, std::vector<size_t>(num_steps, 0));
  for (int r : ctx->DrivenRanks()) {
    std::vector<Task> all_tasks;
    std::vector<void*> all_ptrs;
    for (int s = 0; s < num_steps; ++s) {
      const RankStep& rsx = plan->steps[s][r];
      plan->task_offset[r][s] = all_tasks.size();
      plan->ptr_offset[r][s] = all_ptrs.size();
      all_tasks.insert(all_tasks.end(), rsx.tasks.begin(), rsx.tasks.end());
      for (int slot : rsx.ptr_slots) all_ptrs.push_back(ctx->SlotPtr(r, slot));
    }
    absl::Status cs = CudaStatus(cudaSetDevice(ctx->ranks[r].ordinal), "cudaSetDevice");
    if (!cs.ok()) return cs;
    if (!all_tasks.empty()) {
      void* p = nullptr;
      cs = CudaStatus(cudaMalloc(&p, all_tasks.size() * sizeof(Task)), "cudaMalloc(tasks)");
      if (!cs.ok()) return cs;
      plan->d_tasks[r] = static_cast<Task*>(p);
      cs = CudaStatus(cudaMemcpy(p, all_tasks.data(), all_tasks.size() * sizeof(Task),
                                 cudaMemcpyHostToDevice), "upload tasks");
      if (!cs.ok()) return cs;
    }
    if (!all_ptrs.empty()) {
      void* p = nullptr;
      cs = CudaStatus(cudaMalloc(&p, all_ptrs.size() * sizeof(void*)), "cudaMalloc(ptrs)");
      if (!cs.ok()) return cs;
      plan->d_ptrs[r] = static_cast<void**>(p);
      cs = CudaStatus(cudaMemcpy(p, all_ptrs.data(), all_ptrs.size() * sizeof(void*),
                                 cudaMemcpyHostToDevice), "upload ptrs");
      if (!cs.ok()) return cs;
    }
  }
  *out = plan.release();
  return absl::OkStatus();
}

absl::Status RunPlan(Plan* plan, void* const* device_bufs, void* const* host_bufs,
                     void* const* streams) {
  Context* ctx = plan->ctx;
  if (ctx->is_virtual) return absl::FailedPreconditionError("virtual (planning-only) context cannot run");
  const std::vector<int> driven = ctx->DrivenRanks();
  auto stream_of = [&](size_t i) {
    return streams ? static_cast<cudaStream_t>(streams[i]) : ctx->ranks[driven[i]].stream;
  };
  // Copy-in (user device buffers or host buffers) of every hosted slot.
  if (device_bufs || host_bufs) {
    for (size_t i = 0; i < driven.size(); ++i) {
      const int r = driven[i];
      absl::Status s = CudaStatus(cudaSetDevice(ctx->ranks[r].ordinal), "cudaSetDevice");
      if (!s.ok()) return s;
      for (int d = 0; d < ctx->K; ++d) {
        if (ctx->slot_rank[d] != r) continue;
        const void* src = device_bufs ? device_bufs[d] : host_bufs[d];
        if (!src) return absl::InvalidArgumentError(absl::StrFormat("buffer of slot %d is null", d));
        s = CudaStatus(cudaMemcpyAsync(ctx->SlotPtr(r, d), src, plan->bytes,
                                       device_bufs ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice,
                                       stream_of(i)),
                       "copy-in");
        if (!s.ok()) return s;
      }
    }
  }
  const int S = plan->num_steps;
  const uint32_t piece_bytes = kPieceBytes;
  if (plan->ctas_per_sm == 0 && !driven.empty()) {
    absl::Status st = CudaStatus(cudaSetDevice(ctx->ranks[driven[0]].ordinal), "cudaSetDevice");
    if (!st.ok()) return st;
    plan->ctas_per_sm = MaxResidentCtas(plan->dtype, plan->threads, plan->unroll);
  }
  for (int s = 0; s < S; ++s) {
    for (size_t i = 0; i < driven.size(); ++i) {
      const int r = driven[i];
      const Rank& rank = ctx->ranks[r];
      const RankStep& rsx = plan->steps[s][r];
      StepArgs a{};
      a.tasks = plan->d_tasks[r] ? plan->d_tasks[r] + plan->task_offset[r][s] : nullptr;
      a.ptrs = plan->d_ptrs[r] ? plan->d_ptrs[r] + plan->ptr_offset[r][s] : nullptr;
      a.ntasks = static_cast<uint32_t>(rsx.tasks.size());
      a.npieces = rsx.npieces;
      a.piece_bytes = piece_bytes;
      a.dtype = plan->dtype;
      a.arrive_counter = reinterpret_cast<unsigned int*>(rank.heap + kCounterOffset);
      a.error_flag = reinterpret_cast<int*>(rank.heap + kErrorOffset);
      a.inbox = reinterpret_cast<const uint64_t*>(rank.heap + kInboxOffset);
      a.timeout_ns = ctx->timeout_ns;
      if (ctx->world > 1) {
        for (int q = 0; q < ctx->world; ++q) {
          if (q == r) continue;
          a.signal_ptrs[a.nsignal++] =
              reinterpret_cast<uint64_t*>(rank.view[q] + kInboxOffset) + r;
        }
        for (uint8_t q : rsx.wait) a.wait_ranks[a.nwait++] = q;
        if (s == S - 1) {
          for (int q = 0; q < ctx->world; ++q)
            if (plan->final_wait_bits[r] & (1u << q)) a.final_ranks[a.nfinal++] = static_cast<uint8_t>(q);
        }
      }
      a.epoch_base = reinterpret_cast<uint64_t*>(rank.heap + kEpochOffset);
      a.step = static_cast<uint32_t>(s);
      a.num_steps = static_cast<uint32_t>(S);
      const int resident = plan->ctas_per_sm * rank.sm_count;
      int cap = plan->max_ctas > 0 ? std::min(plan->max_ctas, resident) : resident;
      if (cap <= 0) cap = 148;
      const int grid = std::max(1, std::min<int>(cap, static_cast<int>(rsx.npieces)));
      absl::Status st = CudaStatus(cudaSetDevice(rank.ordinal), "cudaSetDevice");
      if (!st.ok()) return st;
      st = CudaStatus(LaunchStep(a, grid, plan->threads, plan->unroll, stream_of(i)), "step kernel launch");
      if (!st.ok()) return st;
    }
  }
  if (device_bufs || host_bufs) {
    for (size_t i = 0; i < driven.size(); ++i) {
      const int r = driven[i];
      absl::Status s = CudaStatus(cudaSetDevice(ctx->ranks[r].ordinal), "cudaSetDevice");
      if (!s.ok()) return s;
      for (int d = 0; d < ctx->K; ++d) {
        if (ctx->slot_rank[d] != r) continue;
        void* dst = device_bufs ? device_bufs[d] : host_bufs[d];
        s = CudaStatus(cudaMemcpyAsync(dst, ctx->SlotPtr(r, d), plan->bytes,
                                       device_bufs ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                                       stream_of(i)),
                       "copy-out");
        if (!s.ok()) return s;
      }
    }
  }
  return absl::OkStatus();
}

std::string DescribePlan(const Plan& plan) {
  nlohmann::ordered_json doc;
  doc["num_steps"] = plan.num_steps;
  doc["bytes"] = plan.bytes;
  doc["world"] = plan.ctx->world;
  doc["slot_rank"] = plan.ctx->slot_rank;
  nlohmann::ordered_json steps = nlohmann::ordered_json::array();
  for (int s = 0; s < plan.num_steps; ++s) {
    nlohmann::ordered_json ranks = nlohmann::ordered_json::array();
    for (const RankStep& r : plan.steps[s]) {
      nlohmann::ordered_json tasks = nlohmann::ordered_json::array();
      for (const Task& t : r.tasks) {
        std::vector<int> src(r.ptr_slots.begin() + t.ptr_begin, r.ptr_slots.begin() + t.ptr_begin + t.nsrc);
        std::vector<int> dst(r.ptr_slots.begin() + t.ptr_begin + t.nsrc,
                             r.ptr_slots.begin() + t.ptr_begin + t.nsrc + t.ndst);
        tasks.push_back({{"lo", t.lo}, {"hi", t.hi}, {"vec", t.vec}, {"piece_begin", t.piece_begin},
                         {"src", src}, {"dst", dst}});
      }
      std::vector<int> wait(r.wait.begin(), r.wait.end());
      ranks.push_back({{"wait", wait}, {"npieces", r.npieces}, {"tx", r.tx_bytes}, {"rx", r.rx_bytes},
                       {"hbm", r.hbm_bytes}, {"tasks", tasks}});
    }
    steps.push_back({{"ranks", ranks}});
  }
  doc["steps"] = std::move(steps);
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
