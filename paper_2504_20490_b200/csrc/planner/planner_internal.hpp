// hshard-b200 planner internals shared between translation units.
//
// Two geometric tools carry the whole planner:
//   * MixedRadix -- a shard spec read as a row-major mixed-radix number: the
//     device at position i of its group has digit k = (i / stride_k) % radix_k
//     (first entry most significant).  Placement, hsize
//     conversion and collective-group bucketing all read digits through it.
//   * CoverGrid  -- the finest grid that a set of boxes cuts a scope into,
//     walked in row-major cell order with, for every cell, the set of boxes
//     covering it.  Each box is reduced once to per-dimension interval masks,
//     so a cell's cover is the AND of one mask per dimension instead of a
//     containment test per box per cell.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "hshard/annotation.hpp"
#include "hshard/bsr.hpp"

namespace hshard::detail {

class MixedRadix {
 public:
  MixedRadix() = default;
  explicit MixedRadix(std::vector<int> radices);
  static MixedRadix of(const ShardSpec& ds);

  size_t size() const { return radix_.size(); }
  int radix(size_t k) const { return radix_[k]; }
  int digit(int64_t index, size_t k) const {
    return static_cast<int>((index / stride_[k]) % radix_[k]);
  }

 private:
  std::vector<int> radix_;
  std::vector<int64_t> stride_;
};

// Digits of `index` under `radices` (row-major); kept for callers that want
// all digits at once.
std::vector<int> mixed_radix_digits(int64_t index, const std::vector<int>& radices);
std::vector<int> spec_radices(const ShardSpec& ds);

// Sorted, de-duplicated cut positions per dimension, and a row-major walk
// over the cells of the resulting grid (last dimension fastest).  A rank-0
// grid has one (empty) cell; a dimension with fewer than two cuts has none.
using Cuts = std::vector<std::vector<int64_t>>;
void for_each_grid_cell(const Cuts& cuts, const std::function<void(const SliceRegion&)>& fn);

// Set of box indices (bit i = the i-th box given to the CoverGrid).
class CoverSet {
 public:
  CoverSet() = default;
  explicit CoverSet(size_t n) : w_((n + 63) / 64, 0) {}
  void set(size_t i) { w_[i >> 6] |= uint64_t{1} << (i & 63); }
  bool test(size_t i) const { return (w_[i >> 6] >> (i & 63)) & 1; }
  void and_with(const CoverSet& o) {
    for (size_t k = 0; k < w_.size(); ++k) w_[k] &= o.w_[k];
  }
  template <class Fn>
  void each(Fn&& fn) const {  // ascending box index
    for (size_t k = 0; k < w_.size(); ++k)
      for (uint64_t m = w_[k]; m; m &= m - 1) fn(k * 64 + static_cast<size_t>(__builtin_ctzll(m)));
  }

 private:
  std::vector<uint64_t> w_;
};

class CoverGrid {
 public:
  // Cuts: the scope's ends plus every box boundary strictly inside the scope.
  CoverGrid(const SliceRegion& scope, const std::vector<const SliceRegion*>& boxes);

  const Cuts& cuts() const { return cuts_; }
  // fn(cell, cover) for every cell, row-major.
  void walk(const std::function<void(const SliceRegion&, const CoverSet&)>& fn) const;

 private:
  Cuts cuts_;
  std::vector<std::vector<CoverSet>> along_;  // [dim][interval]: boxes spanning it
  size_t nboxes_ = 0;
};

// fuse() over tables shared by several tensors: entry (t, table) contributes
// table's rows labelled as tensor t (no copies); same plan as fuse() over
// relabelled copies of the tables.
BsrPlan fuse_relabelled(const std::vector<std::pair<int, const BsrTable*>>& tables, const Bandwidth& bandwidth);

}  // namespace hshard::detail
