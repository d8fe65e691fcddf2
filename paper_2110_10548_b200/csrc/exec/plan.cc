// Plan compiler: LoweredProgram (CSR) -> per-(phase, rank) task lists.
//
// 1. Replays the reference semantics step by step (redsynth::
//    ApplyCollectiveInPlace, semantics.cc:259-310, folded as RunLowered does,
//    dsl.cc:142-164) to learn which rows every slot holds before each step and
//    to refuse invalid programs with the reference's step/violation.
// 2. Turns every group of every step into owner tasks over row ranges; row r
//    of a slot buffer is elements [floor(rN/K), floor((r+1)N/K)) (SURVEY.md
//    §8(a) a4). One launch per step, variants per step/group:
//      one-shot  small steps whose cross-GPU groups have one member per GPU:
//                sources push flagged 16-byte packets, every destination
//                sums its own result (LayLL);
//      pull      owners load (peer) sources, sum, store (peer) results;
//      push      >= push_min_bytes: sources land the owners' parts in their
//                scratch chunk by chunk behind flags (rotated targets),
//                owners sum locally and store results (LayFlagged);
//      NVLS      AllReduce groups on >= 8 GPUs: multimem.ld_reduce/st.
// 3. Tracks a content id per (slot, row) so copies whose destination already
//    holds bit-identical data (same id) are skipped — the result is the same
//    bits the oracle's unconditional overwrite produces.
// 4. Computes each rank's entry-barrier set per phase (ranks whose memory it
//    touches and their previous-phase writers) and the run's tail barrier.
#include <algorithm>
#include <limits>
#include <map>
#include <memory>
#include <cstdlib>
#include <set>
#include <tuple>

#include "absl/strings/str_format.h"
#include "exec_internal.h"
#include "redsynth/dsl.h"
#include "redsynth/semantics.h"

namespace rs {
namespace {

struct Range {
  uint64_t lo, hi;
};

struct ProtoTask {
  int owner;  // slot whose rank executes the task
  Range range;
  std::vector<Ref> src;  // summation order
  std::vector<Ref> dst;
  int mc = -1;  // >= 0: NVLS through multicast group mc (vector body)
  bool mc_reduce = false;  // NVLS Reduce: ld_reduce, unicast store to dst (else AllReduce)
  bool mc_bcast = false;   // NVLS Broadcast: root's src[0] stored once to the multicast address
  // Push variant (one launch, chunk flags): a landing task (flag_send >= 0)
  // copies its vector body into the owner's memory chunk by chunk and raises
  // flag block `flag_send` per chunk; a reducing task waits for src_flag[i]
  // (-1: no wait) per chunk. Unaligned edges are not pushed: the reducing
  // task's edges pull from edge_src and store to edge_dst.
  int flag_send = -1;
  std::vector<int> src_flag;
  std::vector<Ref> edge_src, edge_dst;
  int wave = 0;  // push variant: pipeline wave (launch order: wave, then landing before reducing)
};

Ref Buf(int slot) { return Ref{slot, -1}; }

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

uint64_t TotalBytes(const std::vector<Range>& ranges) {
  uint64_t t = 0;
  for (const Range& r : ranges) t += r.hi - r.lo;
  return t;
}

// Vector bodies are kVecAlign-aligned (32 B: the one-GPU kernel moves
// 256-bit vectors); owner cuts sit on such offsets, shorter edges become
// scalar tasks.
constexpr uint64_t kVecAlign = 32;

// Splits the concatenation of `ranges` into k consecutive parts of nearly
// equal size whose cut points sit on kVecAlign-byte buffer offsets (or on
// range starts), so owners' vector work stays aligned.
std::vector<std::vector<Range>> SplitEven(const std::vector<Range>& ranges, int k) {
  std::vector<std::vector<Range>> parts(k);
  if (ranges.empty() || k <= 0) return parts;
  const uint64_t total = TotalBytes(ranges);
  auto align = [&](uint64_t c) {
    uint64_t base = 0;
    for (const Range& r : ranges) {
      const uint64_t len = r.hi - r.lo;
      if (c < base + len || (&r == &ranges.back())) {
        const uint64_t b = std::min(r.lo + (c - base), r.hi);
        uint64_t a = b & ~(kVecAlign - 1);
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

// One-shot destination: owner[range] = sum of src[range] in order.
struct LLSpec {
  int owner;
  Range range;
  std::vector<int> src;
};

// Tasks of one program step: push landing tasks (a) and everything else
// (b); both go into the step's single launch, landing tasks first.
struct StepTasks {
  std::vector<ProtoTask> a;  // push landing tasks (empty when nothing pushes)
  std::vector<ProtoTask> b;  // pull tasks and push reducing / fan-out tasks
};

struct Compiler {
  Context* ctx;
  int K;
  int dtype;
  RowGeometry geo;
  std::vector<uint64_t> vid;  // content id of (slot, row)
  uint64_t next_id;
  int next_flag = 0;  // flag blocks of the push variant (per plan)

  Compiler(Context* c, size_t elems, size_t esize, int dt)
      : ctx(c), K(c->K), dtype(dt), geo(elems, c->K, esize), vid(static_cast<size_t>(c->K) * c->K) {
    for (size_t i = 0; i < vid.size(); ++i) vid[i] = i + 1;
    next_id = vid.size() + 1;
  }
  uint64_t& Vid(int d, int r) { return vid[static_cast<size_t>(d) * K + r]; }

  // Push variant: a part is cut into waves of ctx->push_wave_bytes (16-byte
  // aligned cuts); landing and reducing tasks of wave w are laid out before
  // those of wave w+1, so owners reduce (and results leave) while later
  // waves still land — landing and result traffic overlap on every link.
  std::vector<Range> Waves(const Range& r, uint64_t wave_bytes = ~0ull) const {
    const uint64_t w = wave_bytes == ~0ull ? ctx->push_wave_bytes : wave_bytes;
    if (w == 0 || r.hi - r.lo <= w) return {r};
    std::vector<Range> out;
    const uint64_t a = (r.lo + kVecAlign - 1) & ~(kVecAlign - 1);
    uint64_t lo = r.lo;
    for (uint64_t cut = a + w; cut < r.hi; cut += w) {
      out.push_back(Range{lo, cut});
      lo = cut;
    }
    out.push_back(Range{lo, r.hi});
    return out;
  }

  bool SpansRanks(const std::vector<int>& g) const {
    for (int d : g)
      if (ctx->slot_rank[d] != ctx->slot_rank[g[0]]) return true;
    return false;
  }
  // Push needs every sender to land its share in the owner's memory; with
  // senders walking their targets in rotated order (below) it beats pull
  // from ~32 MiB at K=2 and K=4 (profiles/r01_sweep_k4_push.txt).
  bool PushCopies(const std::vector<int>& g, uint64_t bytes, uint64_t min_bytes = ~0ull) const {
    if (min_bytes == ~0ull) min_bytes = ctx->push_min_bytes;
    std::set<int> gpus;
    for (int d : g) gpus.insert(ctx->slot_rank[d]);
    return gpus.size() >= 2 && static_cast<int>(gpus.size()) <= ctx->push_max_gpus && bytes >= min_bytes &&
           bytes > 0;
  }
  bool PushSums(const std::vector<int>& g, uint64_t bytes, uint64_t min_bytes = ~0ull) const {
    return PushCopies(g, bytes, min_bytes) && ctx->scratch_regions >= static_cast<int>(g.size());
  }

  static void Add(std::vector<ProtoTask>& out, int owner, const std::vector<Range>& ranges,
                  const std::vector<Ref>& src, const std::vector<Ref>& dst) {
    for (const Range& r : ranges) out.push_back(ProtoTask{owner, r, src, dst});
  }

  // Sum over group g (order = g) of `parts[j]` owned by members owner_idx[j],
  // results stored to dst_of(j).
  template <typename DstOf>
  void Sums(StepTasks& out, const std::vector<int>& g, const std::vector<int>& owner_idx,
            const std::vector<std::vector<Range>>& parts, bool push, DstOf dst_of,
            uint64_t wave_bytes = ~0ull, const std::vector<uint8_t>& pulled = {}) {
    const int n = static_cast<int>(g.size());
    for (size_t j = 0; j < owner_idx.size(); ++j) {
      const int p = owner_idx[j];
      if (parts[j].empty()) continue;
      std::vector<Ref> src;
      if (!push) {
        for (int m : g) src.push_back(Buf(m));
        Add(out.b, g[p], parts[j], src, dst_of(j));
        continue;
      }
      // (A) every member on another GPU lands its copy of the part in owner
      //     p's scratch region i (members on p's GPU are read in place);
      // (B) owner p waits for each chunk's flags, sums in group order from
      //     local memory and stores.
      const int rp = ctx->slot_rank[g[p]];
      std::vector<Ref> pull_src;
      for (int m : g) pull_src.push_back(Buf(m));
      int wave = 0;
      for (const Range& part : parts[j]) {
        for (const Range& r : Waves(part, wave_bytes)) {
          ProtoTask b{g[p], r, {}, dst_of(j)};
          b.wave = wave;
          for (int i = 0; i < n; ++i) {
            // read in place: the owner's own copy, co-located members, and
            // members marked `pulled` (their copy is loaded remotely by the
            // owner; ready since the step's entry barrier)
            if (i == p || ctx->slot_rank[g[i]] == rp || (i < static_cast<int>(pulled.size()) && pulled[i])) {
              b.src.push_back(Buf(g[i]));
              b.src_flag.push_back(-1);
              continue;
            }
            ProtoTask a{g[i], r, {Buf(g[i])}, {Ref{g[p], i}}};
            a.flag_send = next_flag++;
            a.wave = wave;
            b.src.push_back(Ref{g[p], i});
            b.src_flag.push_back(a.flag_send);
            out.a.push_back(std::move(a));
          }
          b.edge_src = pull_src;
          b.edge_dst = b.dst;
          out.b.push_back(std::move(b));
          ++wave;
        }
      }
    }
  }

  // Copies of rows from their holder to every member whose memory differs
  // (relay: the receivers own slices; a receiver that pulled — or was pushed —
  // its slice fans it out to the other receivers).
  void Copies(StepTasks& out, const std::vector<int>& g,
              const std::vector<std::pair<int, int>>& row_holder) {
    std::map<std::pair<int, std::vector<int>>, std::vector<int>> by_key;
    for (auto [r, h] : row_holder) {
      std::vector<int> recv;
      for (int m : g)
        if (m != h && Vid(m, r) != Vid(h, r)) recv.push_back(m);
      if (!recv.empty()) by_key[{h, recv}].push_back(r);
    }
    // Push only balanced gathers (several holders, e.g. AllGather after a
    // ReduceScatter); a one-to-all copy (Broadcast, AllGather after a Reduce)
    // pulls: measured 15-25 % faster at K=2/K=4 from 128 MiB
    // (profiles/r01_copies_push_vs_pull.txt).
    std::set<int> holders;
    for (auto [r, h] : row_holder) holders.insert(h);
    for (auto& [key, rows] : by_key) {
      const int h = key.first;
      const std::vector<int>& recv = key.second;
      std::sort(rows.begin(), rows.end());
      const std::vector<Range> ranges = geo.Ranges(rows);
      std::vector<int> all = recv;
      all.push_back(h);
      const bool push = holders.size() > 1 && PushCopies(all, TotalBytes(ranges));
      const std::vector<std::vector<Range>> parts = SplitEven(ranges, static_cast<int>(recv.size()));
      for (size_t j = 0; j < recv.size(); ++j) {
        if (parts[j].empty()) continue;
        std::vector<Ref> others;
        for (int m : recv)
          if (m != recv[j]) others.push_back(Buf(m));
        if (push) {
          // (A) the holder lands the part in receiver j's buffer chunk by
          // chunk; (B) receiver j fans each landed chunk out to the others.
          std::vector<Ref> all_dst;
          for (int m : recv) all_dst.push_back(Buf(m));
          int wave = 0;
          for (const Range& part : parts[j]) {
            for (const Range& r : Waves(part)) {
              ProtoTask a{h, r, {Buf(h)}, {Buf(recv[j])}};
              a.flag_send = next_flag++;
              a.wave = wave;
              ProtoTask b{recv[j], r, {Buf(recv[j])}, others};
              b.src_flag = {a.flag_send};
              b.edge_src = {Buf(h)};
              b.edge_dst = all_dst;
              b.wave = wave++;
              out.a.push_back(std::move(a));
              out.b.push_back(std::move(b));
            }
          }
        } else {
          std::vector<Ref> dst;
          for (int m : recv) dst.push_back(Buf(m));
          Add(out.b, recv[j], parts[j], {Buf(h)}, dst);
        }
      }
      for (int r : rows)
        for (int m : recv) Vid(m, r) = Vid(h, r);
    }
  }

  // NVLS applies to AllReduce groups of >= nvls_min_group slots, one per GPU,
  // for floating-point data.
  bool NvlsEligible(const std::vector<int>& g, uint64_t bytes, bool any_dtype = false) const {
    const uint64_t min_bytes = g.size() >= 8 ? ctx->nvls_min_bytes_n8 : ctx->nvls_min_bytes;
    if (!ctx->nvls || (dtype == RS_I32 && !any_dtype) || bytes == 0 || bytes < min_bytes) return false;
    if (static_cast<int>(g.size()) < ctx->nvls_min_group) return false;
    if (ctx->mc_groups.size() >= kMaxMcGroups && !ctx->mc_groups.count(g)) return false;
    std::vector<int> ranks;
    for (int d : g) ranks.push_back(ctx->slot_rank[d]);
    std::sort(ranks.begin(), ranks.end());
    return std::adjacent_find(ranks.begin(), ranks.end()) == ranks.end();
  }

  // One-shot form of a group (LL steps): every destination slot computes its
  // own result from all sources (no owner slicing, no fan-out), so each
  // source's bytes cross NVLink exactly once per receiving GPU. Content ids
  // evolve exactly as in Group().
  void GroupLL(std::vector<LLSpec>& out, const redsynth::StateContext& pre, const std::vector<int>& g,
               redsynth::Collective op) {
    using redsynth::Collective;
    const int n = static_cast<int>(g.size());
    auto add = [&](int owner, const std::vector<Range>& ranges, const std::vector<int>& src) {
      for (const Range& r : ranges) out.push_back(LLSpec{owner, r, src});
    };
    switch (op) {
      case Collective::kAllReduce: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const std::vector<Range> ranges = geo.Ranges(rows);
        for (int m : g) add(m, ranges, g);
        for (int r : rows) {
          const uint64_t id = next_id++;
          for (int m : g) Vid(m, r) = id;
        }
        break;
      }
      case Collective::kReduceScatter: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const int run = n ? static_cast<int>(rows.size()) / n : 0;
        if (run == 0) break;
        for (int m = 0; m < n; ++m)
          add(g[m], geo.Ranges(std::vector<int>(rows.begin() + m * run, rows.begin() + (m + 1) * run)), g);
        for (int m = 0; m < n; ++m)
          for (int i = m * run; i < (m + 1) * run; ++i) Vid(g[m], rows[i]) = next_id++;
        break;
      }
      case Collective::kReduce: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        add(g[0], geo.Ranges(rows), g);
        for (int r : rows) Vid(g[0], r) = next_id++;
        break;
      }
      case Collective::kAllGather:
      case Collective::kBroadcast: {
        std::vector<std::pair<int, int>> row_holder;
        if (op == Collective::kAllGather) {
          for (int r = 0; r < K; ++r)
            for (int m : g)
              if (!pre.state(m).RowEmpty(r)) row_holder.push_back({r, m});
        } else {
          for (int r : HeldRows(pre, g[0])) row_holder.push_back({r, g[0]});
        }
        // (holder, receiver) -> rows, decided on the pre-step content ids.
        std::map<std::pair<int, int>, std::vector<int>> rows_of;
        for (auto [r, h] : row_holder)
          for (int m : g)
            if (m != h && Vid(m, r) != Vid(h, r)) rows_of[{h, m}].push_back(r);
        for (auto& [hm, rows] : rows_of) {
          std::sort(rows.begin(), rows.end());
          add(hm.second, geo.Ranges(rows), {hm.first});
        }
        for (auto& [hm, rows] : rows_of)
          for (int r : rows) Vid(hm.second, r) = Vid(hm.first, r);
        break;
      }
    }
  }

  absl::Status Group(StepTasks& out, const redsynth::StateContext& pre, const std::vector<int>& g,
                     redsynth::Collective op) {
    using redsynth::Collective;
    const int n = static_cast<int>(g.size());
    switch (op) {
      case Collective::kAllReduce: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const std::vector<Range> ranges = geo.Ranges(rows);
        std::vector<int> owners(n);
        for (int i = 0; i < n; ++i) owners[i] = i;
        std::vector<Ref> all;
        for (int m : g) all.push_back(Buf(m));
        int mc = -1;
        if (NvlsEligible(g, TotalBytes(ranges)) && !EnsureMulticast(ctx, g, &mc).ok()) {
          // Every rank sees the same failure (the setup exchanges carry each
          // rank's status), so all fall back to P2P consistently.
          ctx->nvls = false;
          mc = -1;
        }
        if (mc >= 0) {
          const std::vector<std::vector<Range>> parts = SplitEven(ranges, n);
          for (int p = 0; p < n; ++p)
            for (const Range& r : parts[p]) out.b.push_back(ProtoTask{g[p], r, all, all, mc});
        } else {
          Sums(out, g, owners, SplitEven(ranges, n), PushSums(g, TotalBytes(ranges)),
               [&](size_t) { return all; });
        }
        for (int r : rows) {
          const uint64_t id = next_id++;
          for (int m : g) Vid(m, r) = id;
        }
        break;
      }
      case Collective::kReduceScatter: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const int run = n ? static_cast<int>(rows.size()) / n : 0;
        if (run == 0) break;
        std::vector<int> owners(n);
        std::vector<std::vector<Range>> parts(n);
        for (int m = 0; m < n; ++m) {
          owners[m] = m;
          parts[m] = geo.Ranges(std::vector<int>(rows.begin() + m * run, rows.begin() + (m + 1) * run));
        }
        // Pull only: measured faster than push for ReduceScatter at K=2 and
        // K=4 up to 1 GiB (profiles/r01_collectives_vs_nccl.txt).
        Sums(out, g, owners, parts, /*push=*/false, [&](size_t j) { return std::vector<Ref>{Buf(g[j])}; });
        for (int m = 0; m < n; ++m)
          for (int i = m * run; i < (m + 1) * run; ++i) Vid(g[m], rows[i]) = next_id++;
        break;
      }
      case Collective::kReduce: {
        const std::vector<int> rows = HeldRows(pre, g[0]);
        const std::vector<Range> ranges = geo.Ranges(rows);
        // n = 2: the root pulls the other member's data and sums locally —
        // the link carries c one way only (non-root owners would move c both
        // ways and leave all the work to one GPU). n >= 3: the non-roots own
        // slices, so every GPU moves ~c per direction. Pull only (measured
        // faster than push, profiles/r01_collectives_vs_nccl.txt).
        // (Tried for n >= 3: every member owning a slice, root included — no
        // faster; push — slower; owners summing into their scratch behind
        // chunk flags with the root pulling the results — slower.)
        const std::vector<Ref> root{Buf(g[0])};
        int mc = -1;
        int mode = n >= 3 ? ctx->reduce_mode : kReducePull;
        if (mode == kReduceAuto) mode = TotalBytes(ranges) >= ctx->reduce_push_min_bytes ? kReducePush : kReducePull;
        if ((mode == kReduceNvls || mode == kReduceNvlsRoot) && NvlsEligible(g, TotalBytes(ranges)) &&
            !EnsureMulticast(ctx, g, &mc).ok()) {
          ctx->nvls = false;  // consistent P2P fallback on every rank (see AllReduce)
          mc = -1;
        }
        if (mc >= 0) {
          std::vector<Ref> all;
          for (int m : g) all.push_back(Buf(m));
          const int owners_n = mode == kReduceNvlsRoot ? 1 : n;
          const std::vector<std::vector<Range>> parts = SplitEven(ranges, owners_n);
          for (int p = 0; p < owners_n; ++p) {
            for (const Range& r : parts[p]) {
              ProtoTask t{g[p], r, all, root, mc};
              t.mc_reduce = true;
              out.b.push_back(std::move(t));
            }
          }
          for (int r : rows) Vid(g[0], r) = next_id++;
          break;
        }
        std::vector<int> owners;
        if (n == 2) {
          owners.push_back(0);
        } else {
          for (int i = 1; i < n; ++i) owners.push_back(i);
        }
        // kReducePushRootPulled: the owners load the root's copy remotely
        // (the root's SMs issue nothing; its link serves the loads) and
        // every other member lands its copy as in kReducePush.
        std::vector<uint8_t> pulled(n, 0);
        if (mode == kReducePushRootPulled) pulled[0] = 1;
        Sums(out, g, owners, SplitEven(ranges, static_cast<int>(owners.size())),
             (mode == kReducePush || mode == kReducePushRootPulled) && PushSums(g, TotalBytes(ranges), 0),
             [&](size_t) { return root; }, ctx->reduce_wave_bytes, pulled);
        for (int r : rows) Vid(g[0], r) = next_id++;
        break;
      }
      case Collective::kAllGather: {
        std::vector<std::pair<int, int>> row_holder;
        for (int r = 0; r < K; ++r)
          for (int m : g)
            if (!pre.state(m).RowEmpty(r)) row_holder.push_back({r, m});
        Copies(out, g, row_holder);
        break;
      }
      case Collective::kBroadcast: {
        std::vector<std::pair<int, int>> row_holder;
        const std::vector<int> rows = HeldRows(pre, g[0]);
        for (int r : rows) row_holder.push_back({r, g[0]});
        // NVLS: the root stores each byte once to the multicast address and
        // the switch writes every member (bit-exact; any dtype). Only when
        // every member needs every row (no content-id skips).
        bool all_new = true;
        for (int r : rows)
          for (size_t i = 1; i < g.size(); ++i) all_new = all_new && Vid(g[i], r) != Vid(g[0], r);
        const std::vector<Range> ranges = geo.Ranges(rows);
        int mc = -1;
        if (all_new && ctx->nvls_bcast && NvlsEligible(g, TotalBytes(ranges), /*any_dtype=*/true) &&
            !EnsureMulticast(ctx, g, &mc).ok()) {
          ctx->nvls = false;  // consistent P2P fallback on every rank
          mc = -1;
        }
        if (mc >= 0) {
          std::vector<Ref> others;
          for (size_t i = 1; i < g.size(); ++i) others.push_back(Buf(g[i]));
          for (const Range& r : ranges) {
            ProtoTask t{g[0], r, {Buf(g[0])}, others, mc};
            t.mc_bcast = true;
            out.b.push_back(std::move(t));
          }
          for (int r : rows)
            for (size_t i = 1; i < g.size(); ++i) Vid(g[i], r) = Vid(g[0], r);
          break;
        }
        Copies(out, g, row_holder);
        break;
      }
    }
    return absl::OkStatus();
  }
};

void AddTraffic(std::vector<RankStep>& per_rank, const Context& ctx, const ProtoTask& t) {
  const double b = static_cast<double>(t.range.hi - t.range.lo);
  const int o = ctx.slot_rank[t.owner];
  if (t.mc >= 0 && t.mc_bcast) {
    // The root reads its copy and sends it once (tx b); the switch writes
    // every member (rx b each, HBM b each).
    per_rank[o].tx_bytes += b;
    per_rank[o].hbm_bytes += 2 * b;
    for (const Ref& y : t.dst) {
      const int ry = ctx.slot_rank[y.slot];
      per_rank[ry].rx_bytes += b;
      per_rank[ry].hbm_bytes += b;
    }
    return;
  }
  if (t.mc >= 0 && t.mc_reduce) {
    // Switch reads every member's copy (tx b each) and returns the sum to the
    // owner (rx b); the owner stores it to the root (unicast).
    for (const Ref& x : t.src) {
      RankStep& m = per_rank[ctx.slot_rank[x.slot]];
      m.tx_bytes += b;
      m.hbm_bytes += b;
    }
    per_rank[o].rx_bytes += b;
    for (const Ref& y : t.dst) {
      const int ry = ctx.slot_rank[y.slot];
      per_rank[ry].hbm_bytes += b;
      if (ry != o) {
        per_rank[o].tx_bytes += b;
        per_rank[ry].rx_bytes += b;
      }
    }
    return;
  }
  if (t.mc >= 0) {
    // Switch reads every member's copy (tx b each), returns the sum to the
    // owner (rx b); the multicast store leaves the owner (tx b) and lands in
    // every member (rx b).
    for (const Ref& x : t.src) {
      RankStep& m = per_rank[ctx.slot_rank[x.slot]];
      m.tx_bytes += b;
      m.rx_bytes += b;
      m.hbm_bytes += 2 * b;
    }
    per_rank[o].rx_bytes += b;
    per_rank[o].tx_bytes += b;
    return;
  }
  for (const Ref& x : t.src) {
    const int rx = ctx.slot_rank[x.slot];
    per_rank[rx].hbm_bytes += b;
    if (rx != o) {
      per_rank[o].rx_bytes += b;
      per_rank[rx].tx_bytes += b;
    }
  }
  for (const Ref& y : t.dst) {
    const int ry = ctx.slot_rank[y.slot];
    per_rank[ry].hbm_bytes += b;
    if (ry != o) {
      per_rank[o].tx_bytes += b;
      per_rank[ry].rx_bytes += b;
    }
  }
}

Ref FlagRef(int id) { return Ref{id, kFlagRegion}; }  // rank/offset patched per phase
Ref NullRef() { return Ref{-1, kNullRegion}; }

// Push-variant tasks: a landing task is its vector body only; a reducing
// task is its vector body (chunk flags appended to the pointer table) plus
// edges that pull like the default variant.
void LayFlagged(RankStep& rs, const ProtoTask& t, uint64_t chunk, uint64_t recv_piece) {
  const uint64_t a = (t.range.lo + kVecAlign - 1) & ~(kVecAlign - 1);
  const uint64_t b = t.range.hi & ~(kVecAlign - 1);
  auto scalar = [&](uint64_t lo, uint64_t hi) {
    if (hi <= lo || t.edge_dst.empty()) return;
    Task task{};
    task.lo = lo;
    task.hi = hi;
    task.piece_begin = rs.npieces;
    task.ptr_begin = static_cast<uint32_t>(rs.ptr_refs.size());
    task.nsrc = static_cast<uint16_t>(t.edge_src.size());
    task.ndst = static_cast<uint16_t>(t.edge_dst.size());
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.edge_src.begin(), t.edge_src.end());
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.edge_dst.begin(), t.edge_dst.end());
    rs.npieces += 1;
    rs.tasks.push_back(task);
  };
  const bool body = a < b;
  if (t.flag_send >= 0) {
    if (!body) return;
    Task task{};
    task.lo = a;
    task.hi = b;
    task.piece_begin = rs.npieces;
    task.ptr_begin = static_cast<uint32_t>(rs.ptr_refs.size());
    task.nsrc = static_cast<uint16_t>(t.src.size());
    task.ndst = 1;
    task.vec = 1;
    task.mode = kModeFlagSend;
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.src.begin(), t.src.end());
    rs.ptr_refs.push_back(t.dst[0]);
    rs.ptr_refs.push_back(FlagRef(t.flag_send));
    rs.npieces += static_cast<uint32_t>((b - a + chunk - 1) / chunk);
    rs.tasks.push_back(task);
    return;
  }
  if (!body) {  // < 64 bytes: everything pulls
    const uint64_t mid = std::min(std::max(a, t.range.lo), t.range.hi);
    scalar(t.range.lo, mid);
    scalar(mid, t.range.hi);
    return;
  }
  scalar(t.range.lo, a);
  if (!t.dst.empty()) {
    Task task{};
    task.lo = a;
    task.hi = b;
    task.piece_begin = rs.npieces;
    task.ptr_begin = static_cast<uint32_t>(rs.ptr_refs.size());
    task.nsrc = static_cast<uint16_t>(t.src.size());
    task.ndst = static_cast<uint16_t>(t.dst.size());
    task.vec = 1;
    task.mode = kModeFlagRecv;
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.src.begin(), t.src.end());
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.dst.begin(), t.dst.end());
    for (int f : t.src_flag) rs.ptr_refs.push_back(f >= 0 ? FlagRef(f) : NullRef());
    rs.npieces += static_cast<uint32_t>((b - a + recv_piece - 1) / recv_piece);
    rs.tasks.push_back(task);
  }
  scalar(b, t.range.hi);
}

// Places every flag block of a push phase in its owner rank's flag area
// (one uint64 per chunk) and patches the flag references. Returns false if
// a rank's area would overflow.
bool PlaceFlags(const Context& ctx, std::vector<RankStep>& phase) {
  std::map<int, std::pair<int, uint64_t>> where;  // flag id -> (rank, byte offset)
  std::vector<uint64_t> cursor(ctx.world, 0);
  for (int r = 0; r < ctx.world; ++r) {
    for (const Task& t : phase[r].tasks) {
      if (t.mode != kModeFlagSend) continue;
      const Ref& dst = phase[r].ptr_refs[t.ptr_begin + t.nsrc];
      const int id = phase[r].ptr_refs[t.ptr_begin + t.nsrc + t.ndst].slot;
      const int owner_rank = ctx.slot_rank[dst.slot];
      const uint64_t chunks = (t.hi - t.lo + ctx.flag_chunk - 1) / ctx.flag_chunk;
      where[id] = {owner_rank, cursor[owner_rank]};
      cursor[owner_rank] += chunks * sizeof(uint64_t);
    }
  }
  if (!ctx.is_virtual) {
    for (int r = 0; r < ctx.world; ++r)
      if (cursor[r] > ctx.flag_bytes[r]) return false;
  }
  for (RankStep& rs : phase) {
    for (Ref& ref : rs.ptr_refs) {
      if (ref.region != kFlagRegion) continue;
      auto it = where.find(ref.slot);
      if (it == where.end()) return false;
      ref.ll_recv = it->second.first;
      ref.ll_off = static_cast<int64_t>(it->second.second);
    }
  }
  return true;
}

// Appends `t` to its owner rank's phase: vector body + scalar head/tail.
void Lay(RankStep& rs, const ProtoTask& t, uint32_t piece_bytes, uint64_t flag_chunk = 0, uint64_t recv_piece = 0) {
  if (t.flag_send >= 0 || !t.src_flag.empty()) {
    LayFlagged(rs, t, flag_chunk, recv_piece ? recv_piece : flag_chunk);
    return;
  }
  auto push = [&](uint64_t lo, uint64_t hi, bool vec) {
    if (hi <= lo) return;
    Task task{};
    task.lo = lo;
    task.hi = hi;
    task.piece_begin = rs.npieces;
    task.ptr_begin = static_cast<uint32_t>(rs.ptr_refs.size());
    task.vec = vec ? 1u : 0u;
    if (vec && t.mc >= 0 && t.mc_bcast) {
      // NVLS Broadcast body: the root's buffer, then the multicast base.
      task.mode = kModeNvlsBroadcast;
      task.nsrc = 2;
      task.ndst = 0;
      rs.ptr_refs.push_back(t.src[0]);
      rs.ptr_refs.push_back(Ref{t.mc, kMcRegion});
      rs.npieces += static_cast<uint32_t>((hi - lo + piece_bytes - 1) / piece_bytes);
      rs.tasks.push_back(task);
      return;
    }
    if (vec && t.mc >= 0) {
      // NVLS body: one multicast base pointer (unaligned edges stay ordered
      // P2P sums); a Reduce body also lists its unicast destinations.
      task.mode = t.mc_reduce ? kModeNvlsReduce : kModeNvlsAllReduce;
      task.nsrc = 1;
      task.ndst = t.mc_reduce ? static_cast<uint16_t>(t.dst.size()) : 0;
      rs.ptr_refs.push_back(Ref{t.mc, kMcRegion});
      if (t.mc_reduce) rs.ptr_refs.insert(rs.ptr_refs.end(), t.dst.begin(), t.dst.end());
      rs.npieces += static_cast<uint32_t>((hi - lo + piece_bytes - 1) / piece_bytes);
      rs.tasks.push_back(task);
      return;
    }
    task.nsrc = static_cast<uint16_t>(t.src.size());
    task.ndst = static_cast<uint16_t>(t.dst.size());
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.src.begin(), t.src.end());
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.dst.begin(), t.dst.end());
    rs.npieces += vec ? static_cast<uint32_t>((hi - lo + piece_bytes - 1) / piece_bytes) : 1u;
    rs.tasks.push_back(task);
  };
  const uint64_t a = (t.range.lo + kVecAlign - 1) & ~(kVecAlign - 1);
  const uint64_t b = t.range.hi & ~(kVecAlign - 1);
  if (a >= b) {
    // No aligned body: at most 62 bytes, two scalar tasks keep each < 32 B.
    const uint64_t mid = std::min(std::max(a, t.range.lo), t.range.hi);
    push(t.range.lo, mid, false);
    push(mid, t.range.hi, false);
    return;
  }
  push(t.range.lo, a, false);
  push(a, b, true);
  push(b, t.range.hi, false);
}

// Lays a one-shot step into `phase` (one RankStep per rank). Returns false
// (phase untouched) when the step does not fit the LL scheme: a cross-GPU
// group with two members on one GPU, a GPU pair exchanging more than the LL
// budget, or a send whose bytes another task of the step overwrites.
bool LayLL(const Context& ctx, const std::vector<LLSpec>& specs, std::vector<RankStep>& phase) {
  const int R = ctx.world;
  const uint64_t budget = std::min<uint64_t>(ctx.ll_max_bytes, ctx.ll_capacity);
  auto lo8 = [](const Range& r) { return r.lo & ~uint64_t{7}; };
  auto hi8 = [](const Range& r) { return (r.hi + 7) & ~uint64_t{7}; };
  // Payload streams: (sender rank, receiver rank, source slot, lo, hi) -> offset.
  std::map<std::tuple<int, int, int, uint64_t, uint64_t>, uint64_t> stream;
  std::vector<uint64_t> pair_bytes(static_cast<size_t>(R) * R, 0);
  std::vector<uint64_t> sent_bytes(R, 0);
  for (const LLSpec& sp : specs) {
    const int p = ctx.slot_rank[sp.owner];
    int locals = 0;
    for (int x : sp.src) {
      const int q = ctx.slot_rank[x];
      if (q == p) {
        ++locals;
        continue;
      }
      auto key = std::make_tuple(q, p, x, sp.range.lo, sp.range.hi);
      if (stream.count(key)) continue;
      uint64_t& used = pair_bytes[static_cast<size_t>(q) * R + p];
      stream[key] = used;
      used += hi8(sp.range) - lo8(sp.range);
      if (used > budget) return false;
      // Packets double the bytes and go to every receiver separately: a
      // sender's total payload is capped (ll_total_bytes), so wide groups
      // switch to pull earlier.
      sent_bytes[q] += hi8(sp.range) - lo8(sp.range);
      if (sent_bytes[q] > ctx.ll_total_bytes) return false;
    }
    if (locals > 1) return false;
  }
  auto ll_ref = [&](int slot, int recv, int send, uint64_t off, const Range& rg) {
    Ref r{slot, kLLRegion};
    r.ll_recv = recv;
    r.ll_send = send;
    r.ll_off = 2 * static_cast<int64_t>(off) - 2 * static_cast<int64_t>(lo8(rg));
    return r;
  };
  // Receive tasks, one per spec; a source that is itself the owner of the
  // same range (AllReduce) sends its packets from inside its own task, so the
  // value it sends is read before the task overwrites it.
  struct Proto {
    int rank;
    Range range;
    std::vector<Ref> src, dst;
  };
  std::vector<Proto> recv;
  std::map<std::tuple<int, uint64_t, uint64_t>, size_t> fused;  // (owner, lo, hi) -> recv index
  for (const LLSpec& sp : specs) {
    const int p = ctx.slot_rank[sp.owner];
    Proto t{p, sp.range, {}, {Buf(sp.owner)}};
    for (int x : sp.src) {
      const int q = ctx.slot_rank[x];
      t.src.push_back(q == p ? Buf(x) : ll_ref(x, p, q, stream[{q, p, x, sp.range.lo, sp.range.hi}], sp.range));
    }
    if (std::find(sp.src.begin(), sp.src.end(), sp.owner) != sp.src.end())
      fused[{sp.owner, sp.range.lo, sp.range.hi}] = recv.size();
    recv.push_back(std::move(t));
  }
  std::vector<Proto> sends;
  std::map<std::tuple<int, uint64_t, uint64_t>, size_t> send_index;  // (slot, lo, hi) -> sends index
  for (const auto& [key, off] : stream) {
    const auto [q, p, x, lo, hi] = key;
    const Range rg{lo, hi};
    const Ref dst = ll_ref(x, p, q, off, rg);
    auto f = fused.find({x, lo, hi});
    if (f != fused.end()) {
      recv[f->second].dst.push_back(dst);
      continue;
    }
    auto it = send_index.find({x, lo, hi});
    if (it == send_index.end()) {
      it = send_index.emplace(std::make_tuple(x, lo, hi), sends.size()).first;
      sends.push_back(Proto{q, rg, {Buf(x)}, {}});
    }
    sends[it->second].dst.push_back(dst);
  }
  // A separate send reads its slot during the step: nothing may write its
  // range (the padding bytes of edge packets are ignored by the receivers).
  for (const Proto& sd : sends) {
    const int x = sd.src[0].slot;
    for (const LLSpec& sp : specs) {
      if (sp.owner == x && sp.range.lo < sd.range.hi && sd.range.lo < sp.range.hi) return false;
    }
  }
  auto lay = [&](const Proto& t) {
    RankStep& rs = phase[t.rank];
    Task task{};
    task.lo = t.range.lo;
    task.hi = t.range.hi;
    task.piece_begin = rs.npieces;
    task.ptr_begin = static_cast<uint32_t>(rs.ptr_refs.size());
    task.nsrc = static_cast<uint16_t>(t.src.size());
    task.ndst = static_cast<uint16_t>(t.dst.size());
    task.vec = 1;
    task.mode = kModeLL;
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.src.begin(), t.src.end());
    rs.ptr_refs.insert(rs.ptr_refs.end(), t.dst.begin(), t.dst.end());
    const uint64_t span = hi8(t.range) - lo8(t.range);
    rs.npieces += static_cast<uint32_t>((span + kLLPieceBytes - 1) / kLLPieceBytes);
    rs.tasks.push_back(task);
    rs.hbm_bytes += static_cast<double>(t.range.hi - t.range.lo);
    for (const Ref& d : t.dst) {
      if (d.region != kLLRegion) {
        rs.hbm_bytes += static_cast<double>(t.range.hi - t.range.lo);
        continue;
      }
      rs.tx_bytes += 2.0 * static_cast<double>(span);
      phase[d.ll_recv].rx_bytes += 2.0 * static_cast<double>(span);
    }
  };
  for (const Proto& t : sends) lay(t);  // sends first: peers wait on them
  for (const Proto& t : recv) lay(t);
  // Few CTAs: each pays one round trip for all its packets, and a one-CTA
  // launch skips the cross-CTA exit barrier (profiles/r01_ll_sweep_n2.txt).
  uint64_t cta_bytes = 32u << 10;
  if (const char* env = std::getenv("RS_LL_CTA_BYTES")) cta_bytes = std::max<uint64_t>(8, std::strtoull(env, nullptr, 10));
  std::vector<uint64_t> span_bytes(R, 0);
  for (const std::vector<Proto>* list : {&sends, &recv})
    for (const Proto& t : *list) span_bytes[t.rank] += hi8(t.range) - lo8(t.range);
  for (int r = 0; r < R; ++r)
    phase[r].max_grid = static_cast<uint32_t>(std::max<uint64_t>(1, (span_bytes[r] + cta_bytes - 1) / cta_bytes));
  return true;
}

absl::Status Upload(const void* host, size_t bytes, void** dev, const char* what) {
  absl::Status s = CudaStatus(cudaMalloc(dev, bytes), what);
  if (!s.ok()) return s;
  return CudaStatus(cudaMemcpy(*dev, host, bytes, cudaMemcpyHostToDevice), what);
}

}  // namespace

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
  // One GPU (HBM-bound): 8 vectors in flight per thread per source measured
  // +1.7% over 4; across GPUs 4 is as good or better (profiles/r01_tune_*).
  if (ctx->world == 1) plan->unroll = 8;
  // Launch-shape defaults (tuning / A-B runs): RS_THREADS, RS_UNROLL, RS_MAX_CTAS.
  if (const char* v = std::getenv("RS_THREADS")) {
    const int t = std::atoi(v);
    if (t >= 32 && t <= 512 && t % 32 == 0) plan->threads = t;
  }
  if (const char* v = std::getenv("RS_UNROLL")) {
    const int u = std::atoi(v);
    if (u == 4 || u == 8) plan->unroll = u;
  }
  if (const char* v = std::getenv("RS_MAX_CTAS")) plan->max_ctas = std::max(0, std::atoi(v));
  if (const char* v = std::getenv("RS_WIDE_LOADS")) plan->wide_loads = std::atoi(v) != 0;
  if (const char* v = std::getenv("RS_DYNAMIC_PIECES")) plan->dynamic_pieces = std::atoi(v) != 0;
  if (const char* v = std::getenv("RS_PDL")) plan->pdl = std::atoi(v) != 0;
  if (const char* v = std::getenv("RS_PIECE_QUEUE")) plan->piece_queue = std::atoi(v);
  if (const char* v = std::getenv("RS_PUSH_PREFETCH")) plan->push_prefetch = std::atoi(v) != 0;
  if (const char* v = std::getenv("RS_LOCAL_WIDE")) plan->local_wide = std::atoi(v) != 0;
  if (const char* v = std::getenv("RS_VEC256")) plan->vec256 = std::atoi(v);
  if (const char* v = std::getenv("RS_REMOTE256")) plan->remote256 = std::atoi(v) != 0;
  {
    const uint64_t rp = ctx->recv_piece_bytes;
    plan->recv_piece = static_cast<uint32_t>(rp >= 16 && rp % 16 == 0 && ctx->flag_chunk % rp == 0 ? rp : ctx->flag_chunk);
  }

  // 2./3. Tasks per step, laid out into one launch phase per step.
  Compiler comp(ctx, elems, es, dtype);
  const int R = ctx->world;
  std::vector<std::vector<int>> gidx(num_steps, std::vector<int>(K, -1));  // -1 = idle
  for (int s = 0; s < num_steps; ++s) {
    StepTasks tasks;
    const redsynth::CollectiveStep& step = lowered.steps[s];
    for (size_t gi = 0; gi < step.groups.size(); ++gi)
      for (int d : step.groups[gi]) gidx[s][d] = static_cast<int>(gi);
    // One-shot (LL) attempt: cross-GPU groups as LLSpecs, GPU-local groups as
    // ordinary tasks, all in one launch; on any misfit roll back the content
    // ids and take the pull / push / NVLS path.
    if (R > 1 && ctx->ll_capacity > 0 && ctx->ll_max_bytes > 0) {
      const std::vector<uint64_t> saved_vid = comp.vid;
      const uint64_t saved_next = comp.next_id;
      std::vector<LLSpec> specs;
      StepTasks local;
      for (const std::vector<int>& g : step.groups) {
        if (comp.SpansRanks(g)) {
          comp.GroupLL(specs, pre[s], g, step.op);
        } else {
          absl::Status gs = comp.Group(local, pre[s], g, step.op);
          if (!gs.ok()) return gs;
        }
      }
      std::vector<RankStep> phase(R);
      bool ok = local.a.empty() && !specs.empty();
      if (ok) {
        for (int r = 0; r < R; ++r) phase[r].piece_bytes = kLLPieceBytes;
        ok = LayLL(*ctx, specs, phase);
      }
      if (ok) {
        for (const ProtoTask& t : local.b) {
          AddTraffic(phase, *ctx, t);
          Lay(phase[ctx->slot_rank[t.owner]], t, kLLPieceBytes);
        }
        plan->phases.push_back(std::move(phase));
        plan->phase_step.push_back(s);
        plan->phase_ll.push_back(1);
        continue;
      }
      comp.vid = saved_vid;
      comp.next_id = saved_next;
    }
    for (size_t gi = 0; gi < step.groups.size(); ++gi) {
      absl::Status gs = comp.Group(tasks, pre[s], step.groups[gi], step.op);
      if (!gs.ok()) return gs;
    }
    // One launch: push landing tasks first (every CTA sends before it waits
    // for chunks), then the reducing / pull tasks.
    // Order: per push wave, its landing tasks (each sender walking the
    // receiving GPUs starting after itself, so at any moment the GPUs push
    // into different peers rather than all into one), then its reducing /
    // fan-out tasks; tasks without flags (pull) last. Every CTA meets a
    // wave's landing pieces before that wave's reducing pieces, so the waits
    // cannot deadlock (all CTAs of a launch are resident).
    std::vector<ProtoTask> list = std::move(tasks.a);
    list.insert(list.end(), tasks.b.begin(), tasks.b.end());
    // A wave's reducing pieces are handed out after the landing pieces of
    // wave_lag later waves (still deadlock-free: landing pieces never wait).
    const int lag = ctx->wave_lag;
    auto order_key = [&](const ProtoTask& t) {
      if (t.flag_send >= 0) {
        const int from = ctx->slot_rank[t.owner];
        return std::make_tuple(t.wave, 0, (ctx->slot_rank[t.dst[0].slot] - from + R) % R);
      }
      if (!t.src_flag.empty()) return std::make_tuple(t.wave + lag, 1, 0);
      return std::make_tuple(std::numeric_limits<int>::max(), 2, 0);
    };
    std::stable_sort(list.begin(), list.end(),
                     [&](const ProtoTask& x, const ProtoTask& y) { return order_key(x) < order_key(y); });
    plan->phases.emplace_back(R);
    plan->phase_step.push_back(s);
    plan->phase_ll.push_back(0);
    // Piece size per rank: enough pieces to occupy ~2 CTAs per SM (memory
    // parallelism for remote loads), between 4 KiB and kPieceBytes.
    std::vector<uint64_t> rank_bytes(R, 0);
    for (const ProtoTask& t : list) rank_bytes[ctx->slot_rank[t.owner]] += t.range.hi - t.range.lo;
    uint32_t max_piece = kPieceBytes;  // RS_MAX_PIECE (A/B; power of two, 16 KiB .. 1 MiB)
    if (const char* v = std::getenv("RS_MAX_PIECE")) {
      const uint32_t m = static_cast<uint32_t>(std::strtoul(v, nullptr, 10));
      if (m >= (16u << 10) && m <= (1u << 20) && (m & (m - 1)) == 0) max_piece = m;
    }
    for (int r = 0; r < R; ++r) {
      const uint64_t sms = ctx->ranks[r].sm_count > 0 ? ctx->ranks[r].sm_count : kDefaultSmCount;
      uint32_t pb = 4u << 10;
      while (pb < max_piece && rank_bytes[r] / pb > 2 * sms) pb <<= 1;
      plan->phases.back()[r].piece_bytes = pb;
      // Push reductions: 64 KiB pieces keep every CTA busy when results fan
      // out to n members (AllReduce, AllGather); a Reduce's owners store one
      // result each and run best on whole chunks (K=4 1 GiB 2,186 -> 1,812 us,
      // profiles/r02_reduce_variants_k4.txt).
      plan->phases.back()[r].recv_piece = step.op == Collective::kReduce ? static_cast<uint32_t>(ctx->flag_chunk)
                                                                         : plan->recv_piece;
    }
    for (const ProtoTask& t : list) {
      AddTraffic(plan->phases.back(), *ctx, t);
      RankStep& rs = plan->phases.back()[ctx->slot_rank[t.owner]];
      Lay(rs, t, rs.piece_bytes, ctx->flag_chunk, rs.recv_piece);
    }
    if (comp.next_flag > 0 && !PlaceFlags(*ctx, plan->phases.back())) {
      return absl::InternalError("push variant: flag area overflow");
    }
  }

  // Distinct peer GPUs each rank's tasks address per phase (launch shape).
  for (std::vector<RankStep>& phase : plan->phases) {
    for (int r = 0; r < R; ++r) {
      std::set<int> peers;
      for (const Ref& ref : phase[r].ptr_refs) {
        if (ref.region == kMcRegion || ref.region == kNullRegion) continue;
        const int q = (ref.region == kLLRegion || ref.region == kFlagRegion) ? ref.ll_recv : ctx->slot_rank[ref.slot];
        if (q != r) peers.insert(q);
      }
      phase[r].remote_peers = static_cast<int>(peers.size());
    }
  }

  // 4. Barrier sets (phases of one step share its groups).
  const int P = plan->num_phases();
  auto group_of = [&](int ph, int d) -> std::vector<int> {
    if (ph < 0) return {d};
    const int s = plan->phase_step[ph];
    if (gidx[s][d] < 0) return {d};
    return lowered.steps[s].groups[gidx[s][d]];
  };
  plan->final_wait_bits.assign(R, 0);
  for (int ph = 0; ph < P; ++ph) {
    for (int r = 0; r < R; ++r) {
      std::set<int> wait;
      for (int d = 0; d < K; ++d) {
        if (ctx->slot_rank[d] != r) continue;
        for (int q : group_of(ph, d))
          for (int p : group_of(ph - 1, q)) wait.insert(ctx->slot_rank[p]);
      }
      wait.erase(r);
      plan->phases[ph][r].wait.assign(wait.begin(), wait.end());
    }
  }
  // A one-shot last phase writes only its own GPU's slots: no tail wait.
  if (P > 0 && !plan->phase_ll[P - 1]) {
    for (int d = 0; d < K; ++d) {
      const int r = ctx->slot_rank[d];
      for (int p : group_of(P - 1, d)) {
        const int q = ctx->slot_rank[p];
        if (q != r) plan->final_wait_bits[r] |= static_cast<uint8_t>(1u << q);
      }
    }
  }

  // A one-shot phase right after another one-shot phase waits one epoch
  // less: nobody wrote or reads its ranks' slots remotely in the previous
  // phase, so it only has to know that its receivers consumed the packets
  // of two phases ago (same parity region), i.e. finished phase t-2.
  plan->phase_lag.assign(P, 0);
  for (int ph = 1; ph < P; ++ph) plan->phase_lag[ph] = plan->phase_ll[ph] && plan->phase_ll[ph - 1] ? 1 : 0;
  // End-of-phase epochs nobody waits for are not published (the exit fence
  // is most of a small step's cost): phase ph's epoch is awaited by phase
  // ph+1 (lag 0) or ph+2 (lag 1) entry sets, or, for the last phase, by the
  // tail waits.
  for (int ph = 0; ph < P; ++ph) {
    for (int r = 0; r < R; ++r) {
      bool needed = ph + 1 == P && [&] {
        for (int q = 0; q < R; ++q)
          if (q != r && ((plan->final_wait_bits[q] >> r) & 1u)) return true;
        return false;
      }();
      for (int t = ph + 1; t < P && t <= ph + 2 && !needed; ++t) {
        if (t - plan->phase_lag[t] - 1 != ph) continue;
        for (int q = 0; q < R && !needed; ++q) {
          if (q == r) continue;
          const std::vector<uint8_t>& w = plan->phases[t][q].wait;
          needed = std::find(w.begin(), w.end(), static_cast<uint8_t>(r)) != w.end();
        }
      }
      plan->phases[ph][r].signal_done = needed;
    }
  }

  // Device copies for every rank this process drives.
  plan->d_tasks.assign(R, nullptr);
  plan->d_ptrs.assign(R, nullptr);
  plan->task_offset.assign(R, std::vector<size_t>(P, 0));
  plan->ptr_offset.assign(R, std::vector<size_t>(P, 0));
  for (int r : ctx->DrivenRanks()) {
    std::vector<Task> all_tasks;
    std::vector<void*> all_ptrs;
    for (int ph = 0; ph < P; ++ph) {
      const RankStep& rsx = plan->phases[ph][r];
      plan->task_offset[r][ph] = all_tasks.size();
      plan->ptr_offset[r][ph] = all_ptrs.size();
      all_tasks.insert(all_tasks.end(), rsx.tasks.begin(), rsx.tasks.end());
      for (const Ref& ref : rsx.ptr_refs) all_ptrs.push_back(ctx->RefPtr(r, ref));
    }
    absl::Status cs = CudaStatus(cudaSetDevice(ctx->ranks[r].ordinal), "cudaSetDevice");
    if (!cs.ok()) return cs;
    if (!all_tasks.empty()) {
      void* p = nullptr;
      cs = Upload(all_tasks.data(), all_tasks.size() * sizeof(Task), &p, "upload tasks");
      plan->d_tasks[r] = static_cast<Task*>(p);
      if (!cs.ok()) return cs;
    }
    if (!all_ptrs.empty()) {
      void* p = nullptr;
      cs = Upload(all_ptrs.data(), all_ptrs.size() * sizeof(void*), &p, "upload pointers");
      plan->d_ptrs[r] = static_cast<void**>(p);
      if (!cs.ok()) return cs;
    }
  }
  *out = plan.release();
  return absl::OkStatus();
}

}  // namespace rs
