// hshard-b200 planner: mixed-radix digits and covered grids (see
// planner_internal.hpp).
#include <algorithm>

#include "planner_internal.hpp"

namespace hshard::detail {

MixedRadix::MixedRadix(std::vector<int> radices) : radix_(std::move(radices)), stride_(radix_.size(), 1) {
  for (size_t k = radix_.size(); k-- > 1;) stride_[k - 1] = stride_[k] * radix_[k];
}

MixedRadix MixedRadix::of(const ShardSpec& ds) { return MixedRadix(spec_radices(ds)); }

std::vector<int> spec_radices(const ShardSpec& ds) {
  std::vector<int> r(ds.entries.size());
  std::transform(ds.entries.begin(), ds.entries.end(), r.begin(), [](const ShardEntry& e) { return e.count; });
  return r;
}

std::vector<int> mixed_radix_digits(int64_t index, const std::vector<int>& radices) {
  const MixedRadix mr(radices);
  std::vector<int> d(radices.size());
  for (size_t k = 0; k < d.size(); ++k) d[k] = mr.digit(index, k);
  return d;
}

namespace {

// Row-major odometer over per-dimension interval counts; calls fn(pos, first_changed_dim).
template <class Fn>
void odometer(const std::vector<size_t>& extent, Fn&& fn) {
  const size_t rank = extent.size();
  for (size_t n : extent)
    if (n == 0) return;
  std::vector<size_t> pos(rank, 0);
  size_t changed = 0;
  for (;;) {
    fn(pos, changed);
    size_t d = rank;
    while (d > 0 && ++pos[d - 1] == extent[d - 1]) pos[--d] = 0;
    if (d == 0) return;
    changed = d - 1;
  }
}

std::vector<size_t> interval_counts(const Cuts& cuts) {
  std::vector<size_t> n(cuts.size());
  for (size_t d = 0; d < cuts.size(); ++d) n[d] = cuts[d].size() < 2 ? 0 : cuts[d].size() - 1;
  return n;
}

}  // namespace

void for_each_grid_cell(const Cuts& cuts, const std::function<void(const SliceRegion&)>& fn) {
  SliceRegion cell;
  cell.bounds.resize(cuts.size());
  odometer(interval_counts(cuts), [&](const std::vector<size_t>& pos, size_t changed) {
    for (size_t d = changed; d < pos.size(); ++d) cell.bounds[d] = {cuts[d][pos[d]], cuts[d][pos[d] + 1]};
    fn(cell);
  });
}

CoverGrid::CoverGrid(const SliceRegion& scope, const std::vector<const SliceRegion*>& boxes)
    : cuts_(scope.bounds.size()), along_(scope.bounds.size()), nboxes_(boxes.size()) {
  for (size_t d = 0; d < cuts_.size(); ++d) {
    const int64_t lo = scope.bounds[d][0], hi = scope.bounds[d][1];
    std::vector<int64_t>& c = cuts_[d];
    c = {lo, hi};
    for (const SliceRegion* b : boxes)
      for (int64_t v : b->bounds[d])
        if (lo < v && v < hi) c.push_back(v);
    std::sort(c.begin(), c.end());
    c.erase(std::unique(c.begin(), c.end()), c.end());
    // a box spans interval [c_i, c_i+1) along d iff its bounds enclose it
    const size_t n = c.size() < 2 ? 0 : c.size() - 1;
    along_[d].assign(n, CoverSet(nboxes_));
    for (size_t b = 0; b < boxes.size(); ++b) {
      const auto& bb = boxes[b]->bounds[d];
      const size_t first = std::lower_bound(c.begin(), c.end(), bb[0]) - c.begin();
      for (size_t i = first; i < n && c[i + 1] <= bb[1]; ++i)
        if (bb[0] <= c[i]) along_[d][i].set(b);
    }
  }
}

void CoverGrid::walk(const std::function<void(const SliceRegion&, const CoverSet&)>& fn) const {
  const size_t rank = cuts_.size();
  SliceRegion cell;
  cell.bounds.resize(rank);
  CoverSet all(nboxes_);
  for (size_t b = 0; b < nboxes_; ++b) all.set(b);
  if (rank == 0) {
    fn(cell, all);
    return;
  }
  // prefix[d] = cover of dims 0..d at the current position
  std::vector<CoverSet> prefix(rank, all);
  odometer(interval_counts(cuts_), [&](const std::vector<size_t>& pos, size_t changed) {
    for (size_t d = changed; d < rank; ++d) {
      cell.bounds[d] = {cuts_[d][pos[d]], cuts_[d][pos[d] + 1]};
      prefix[d] = d ? prefix[d - 1] : all;
      prefix[d].and_with(along_[d][pos[d]]);
    }
    fn(cell, prefix[rank - 1]);
  });
}

}  // namespace hshard::detail
