// Parallelism specs and placement matrices.
// Behaviour follows /root/reference/proj/src/placement.cc:28-158: the same
// validation messages, and the same output set (every grid whose rows
// multiply to the axis sizes and whose columns multiply to the level
// cardinalities) in the same order (ascending row-major flat()).
#include "redsynth/placement.h"

#include <algorithm>
#include <cstdint>
#include <string>

#include "absl/status/status.h"
#include "absl/strings/str_format.h"

namespace redsynth {

absl::Status ValidateSpec(const ParallelismSpec& spec, const SystemModel& system) {
  if (spec.axes.empty()) return absl::InvalidArgumentError("parallelism axes must be nonempty");
  int64_t product = 1;
  for (int size : spec.axes) {
    if (size < 1) return absl::InvalidArgumentError("axis sizes must be >= 1");
    product *= size;
  }
  if (product != system.device_count()) {
    return absl::InvalidArgumentError(
        absl::StrFormat("product of axes (%d) must equal the device count (%d)", product,
                        system.device_count()));
  }
  if (spec.reduction_axes.empty()) {
    return absl::InvalidArgumentError("reduction axes must be nonempty");
  }
  int previous = -1;
  for (int axis : spec.reduction_axes) {
    if (axis < 0 || axis >= static_cast<int>(spec.axes.size())) {
      return absl::InvalidArgumentError(absl::StrFormat("reduction axis %d out of range", axis));
    }
    if (axis <= previous) {
      return absl::InvalidArgumentError("reduction axes must be sorted and unique");
    }
    previous = axis;
  }
  return absl::OkStatus();
}

ParallelismMatrix ParallelismMatrix::FromRows(const std::vector<std::vector<int>>& rows) {
  const int axes = static_cast<int>(rows.size());
  const int levels = static_cast<int>(rows.front().size());
  ParallelismMatrix m(axes, levels);
  for (int a = 0; a < axes; ++a)
    for (int l = 0; l < levels; ++l) m.set_factor(a, l, rows[a][l]);
  return m;
}

std::vector<int> ParallelismMatrix::AxisRow(int axis) const {
  auto first = factors_.begin() + static_cast<std::ptrdiff_t>(axis) * num_levels_;
  return std::vector<int>(first, first + num_levels_);
}

std::string ParallelismMatrix::ToString() const {
  std::string out = "[";
  for (int a = 0; a < num_axes_; ++a) {
    if (a) out += ",";
    out += "[";
    for (int l = 0; l < num_levels_; ++l) {
      if (l) out += ",";
      out += std::to_string(factor(a, l));
    }
    out += "]";
  }
  out += "]";
  return out;
}

namespace {

// Depth-first over cells in column-major order (level, then axis). `remaining`
// holds, per axis, the part of its size not yet placed; `column_left` the
// part of the current level's cardinality not yet assigned.
class GridSearch {
 public:
  GridSearch(const SystemModel& system, const std::vector<int>& axes)
      : system_(system),
        num_axes_(static_cast<int>(axes.size())),
        remaining_(axes.begin(), axes.end()),
        grid_(num_axes_, system.num_levels()) {}

  std::vector<ParallelismMatrix> Run() {
    Visit(0, 0, system_.num_levels() > 0 ? system_.level(0).cardinality : 1);
    return std::move(found_);
  }

 private:
  void Visit(int level, int axis, int column_left) {
    if (level == system_.num_levels()) {
      for (int64_t r : remaining_) {
        if (r != 1) return;
      }
      found_.push_back(grid_);
      return;
    }
    if (axis == num_axes_) {
      if (column_left != 1) return;
      const int next = level + 1;
      Visit(next, 0, next < system_.num_levels() ? system_.level(next).cardinality : 1);
      return;
    }
    for (int f = 1; f <= column_left; ++f) {
      if (column_left % f != 0 || remaining_[axis] % f != 0) continue;
      remaining_[axis] /= f;
      grid_.set_factor(axis, level, f);
      Visit(level, axis + 1, column_left / f);
      remaining_[axis] *= f;
    }
    grid_.set_factor(axis, level, 1);
  }

  const SystemModel& system_;
  int num_axes_;
  std::vector<int64_t> remaining_;
  ParallelismMatrix grid_;
  std::vector<ParallelismMatrix> found_;
};

}  // namespace

absl::StatusOr<std::vector<ParallelismMatrix>> EnumerateMatrices(const SystemModel& system,
                                                                 const ParallelismSpec& spec) {
  absl::Status valid = ValidateSpec(spec, system);
  if (!valid.ok()) return valid;
  std::vector<ParallelismMatrix> grids = GridSearch(system, spec.axes).Run();
  std::sort(grids.begin(), grids.end(),
            [](const ParallelismMatrix& x, const ParallelismMatrix& y) { return x.flat() < y.flat(); });
  grids.erase(std::unique(grids.begin(), grids.end()), grids.end());
  return grids;
}

}  // namespace redsynth
