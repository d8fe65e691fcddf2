// The reduction-program DSL: group derivation, lowering to physical devices,
// the symbolic executor and the text grammar.
// Behaviour follows /root/reference/proj/src/dsl.cc: DeriveGroups :27-92,
// Lower :94-133, RunLowered :142-164, PrettyPrint/ParseProgram :166-275.
#include "redsynth/dsl.h"

#include <algorithm>

#include "absl/status/status.h"
#include "absl/strings/str_format.h"
#include "absl/strings/str_join.h"
#include "absl/strings/str_split.h"

namespace redsynth {

absl::StatusOr<std::vector<std::vector<int>>> DeriveGroups(const SynthesisHierarchy& hierarchy,
                                                           int slice, Form form) {
  const int last = hierarchy.num_levels() - 1;
  if (slice < 0 || slice > last) {
    return absl::InvalidArgumentError(absl::StrFormat("slice level %d out of range", slice));
  }
  const bool keyed = form.kind != Form::kInsideGroup;
  if (keyed && (form.ancestor < 0 || form.ancestor >= slice)) {
    return absl::InvalidArgumentError(absl::StrFormat(
        "form level %d must be a strict ancestor of slice %d", form.ancestor, slice));
  }
  const std::vector<int> card = hierarchy.cardinalities();
  // below[t]: devices under one instance of level t.
  std::vector<int> below(last + 1, 1);
  for (int t = last - 1; t >= 0; --t) below[t] = below[t + 1] * card[t + 1];
  auto product = [&](int from, int to) {  // card[from..to]
    int p = 1;
    for (int t = from; t <= to; ++t) p *= card[t];
    return p;
  };

  std::vector<std::vector<int>> groups;
  if (!keyed) {
    // One group per instance of the slice level: its whole subtree.
    const int size = below[slice];
    if (size <= 1) return absl::FailedPreconditionError("instruction groups only single devices");
    const int count = product(0, slice);
    groups.resize(count, std::vector<int>(size));
    for (int p = 0; p < count; ++p)
      for (int m = 0; m < size; ++m) groups[p][m] = p * size + m;
    return groups;
  }
  // Parallel/Master: members vary the digits of levels ancestor+1..slice;
  // the prefix (levels 0..ancestor) and suffix (below the slice) stay fixed.
  const int a = form.ancestor;
  const int size = product(a + 1, slice);
  if (size <= 1) return absl::FailedPreconditionError("instruction groups only single devices");
  const int prefixes = product(0, a);
  const int suffixes = below[slice];
  const int suffix_end = form.kind == Form::kMaster ? 1 : suffixes;
  for (int p = 0; p < prefixes; ++p) {
    for (int s = 0; s < suffix_end; ++s) {
      std::vector<int> g(size);
      for (int m = 0; m < size; ++m) g[m] = p * below[a] + m * below[slice] + s;
      groups.push_back(std::move(g));
    }
  }
  return groups;
}

absl::StatusOr<LoweredProgram> Lower(const Program& program, const SynthesisHierarchy& hierarchy,
                                     const HierarchyEmbedding& embedding) {
  LoweredProgram lowered;
  lowered.steps.reserve(program.instructions.size());
  for (const ReductionInstruction& ins : program.instructions) {
    absl::StatusOr<std::vector<std::vector<int>>> pattern =
        DeriveGroups(hierarchy, ins.slice, ins.form);
    if (!pattern.ok()) return pattern.status();
    CollectiveStep step;
    step.op = ins.op;
    step.groups.reserve(static_cast<size_t>(embedding.num_assignments()) * pattern->size());
    for (int asg = 0; asg < embedding.num_assignments(); ++asg) {
      for (const std::vector<int>& g : *pattern) {
        std::vector<int> physical(g.size());
        std::transform(g.begin(), g.end(), physical.begin(),
                       [&](int idx) { return embedding.PhysicalOf(idx, asg); });
        step.groups.push_back(std::move(physical));
      }
    }
    std::sort(step.groups.begin(), step.groups.end(),
              [](const std::vector<int>& x, const std::vector<int>& y) { return x.front() < y.front(); });
    lowered.steps.push_back(std::move(step));
  }
  return lowered;
}

absl::StatusOr<LoweredProgram> Lower(const Program& program, const ParallelismMatrix& matrix,
                                     std::span<const int> reduction_axes,
                                     const SystemModel& system) {
  const SynthesisHierarchy h =
      BuildHierarchy(matrix, reduction_axes, system, HierarchyKind::kReductionAxis);
  return Lower(program, h, HierarchyEmbedding(h, matrix, system));
}

std::string StepFailure::Describe() const {
  return absl::StrFormat("step %d: %s over devices {%s}: %s", step, ToString(op),
                         absl::StrJoin(group, ","), ToString(violation));
}

absl::StatusOr<StateContext> RunLowered(const LoweredProgram& lowered, int k,
                                        StepFailure* failure) {
  StateContext ctx = InitialContext(k);
  for (size_t s = 0; s < lowered.steps.size(); ++s) {
    const CollectiveStep& step = lowered.steps[s];
    if (step.groups.empty()) {
      return absl::InvalidArgumentError(
          absl::StrFormat("step %d has no device groups", static_cast<int>(s)));
    }
    for (const std::vector<int>& g : step.groups) {
      const RuleViolation v = ApplyCollectiveInPlace(ctx, g, step.op);
      if (v == RuleViolation::kNone) continue;
      StepFailure what;
      what.step = static_cast<int>(s);
      what.op = step.op;
      what.violation = v;
      what.group = g;
      if (failure) *failure = what;
      return absl::FailedPreconditionError(what.Describe());
    }
  }
  return ctx;
}

std::string PrettyPrint(const ReductionInstruction& ins, const SynthesisHierarchy& hierarchy) {
  std::string form = "InsideGroup";
  if (ins.form.kind == Form::kParallel) {
    form = absl::StrFormat("Parallel(%s)", hierarchy.levels[ins.form.ancestor].label);
  } else if (ins.form.kind == Form::kMaster) {
    form = absl::StrFormat("Master(%s)", hierarchy.levels[ins.form.ancestor].label);
  }
  return absl::StrFormat("Slice(%s) %s %s", hierarchy.levels[ins.slice].label, form,
                         ToString(ins.op));
}

std::string PrettyPrint(const Program& program, const SynthesisHierarchy& hierarchy) {
  std::string text;
  for (size_t i = 0; i < program.instructions.size(); ++i) {
    if (i) text += "; ";
    text += PrettyPrint(program.instructions[i], hierarchy);
  }
  return text;
}

namespace {

absl::StatusOr<int> LevelByLabel(const SynthesisHierarchy& hierarchy, std::string_view label) {
  const int index = hierarchy.LevelIndexOf(label);
  if (index >= 0) return index;
  return absl::InvalidArgumentError(absl::StrFormat("unknown hierarchy level '%s'", label));
}

// "Name(inner)" -> inner, or nullopt-like empty flag when the shape is wrong.
bool Unwrap(std::string_view token, std::string_view name, std::string_view* inner) {
  if (token.size() < name.size() + 2 || token.substr(0, name.size()) != name ||
      token[name.size()] != '(' || token.back() != ')') {
    return false;
  }
  *inner = token.substr(name.size() + 1, token.size() - name.size() - 2);
  return true;
}

absl::StatusOr<ReductionInstruction> ParseOne(const std::string& text,
                                              const SynthesisHierarchy& hierarchy) {
  const std::vector<std::string> tok = absl::StrSplit(text, ' ', absl::SkipEmpty());
  if (tok.size() != 3) {
    return absl::InvalidArgumentError(
        absl::StrFormat("expected 'Slice(level) form op', got '%s'", text));
  }
  ReductionInstruction ins;
  std::string_view inner;
  if (!Unwrap(tok[0], "Slice", &inner)) {
    return absl::InvalidArgumentError(absl::StrFormat("expected 'Slice(level)', got '%s'", tok[0]));
  }
  absl::StatusOr<int> slice = LevelByLabel(hierarchy, inner);
  if (!slice.ok()) return slice.status();
  ins.slice = *slice;

  if (tok[1] == "InsideGroup") {
    ins.form = Form::InsideGroup();
  } else {
    const bool parallel = Unwrap(tok[1], "Parallel", &inner);
    if (!parallel && !Unwrap(tok[1], "Master", &inner)) {
      return absl::InvalidArgumentError(absl::StrFormat("unknown form '%s'", tok[1]));
    }
    absl::StatusOr<int> anc = LevelByLabel(hierarchy, inner);
    if (!anc.ok()) return anc.status();
    ins.form = parallel ? Form::Parallel(*anc) : Form::Master(*anc);
    if (ins.form.ancestor >= ins.slice) {
      return absl::InvalidArgumentError(absl::StrFormat(
          "form level must be a strict ancestor of the slice in '%s'", text));
    }
  }
  absl::StatusOr<Collective> op = ParseCollective(tok[2]);
  if (!op.ok()) return op.status();
  ins.op = *op;
  return ins;
}

}  // namespace

absl::StatusOr<Program> ParseProgram(std::string_view text, const SynthesisHierarchy& hierarchy) {
  Program program;
  const std::vector<std::string> parts = absl::StrSplit(text, ';');
  for (const std::string& raw : parts) {
    const size_t b = raw.find_first_not_of(' ');
    if (b == std::string::npos) continue;
    const size_t e = raw.find_last_not_of(' ');
    absl::StatusOr<ReductionInstruction> ins = ParseOne(raw.substr(b, e - b + 1), hierarchy);
    if (!ins.ok()) return ins.status();
    program.instructions.push_back(*ins);
  }
  if (program.instructions.empty()) {
    return absl::InvalidArgumentError("program must have >= 1 instruction");
  }
  return program;
}

}  // namespace redsynth
