// hshard-b200 planner internals shared between translation units.
#pragma once

#include <cstdint>
#include <functional>
#include <vector>

#include "hshard/annotation.hpp"

namespace hshard::detail {

// Row-major mixed-radix digits of `index` (first radix most significant).
std::vector<int> mixed_radix_digits(int64_t index, const std::vector<int>& radices);
std::vector<int> spec_radices(const ShardSpec& ds);

// Sorted, de-duplicated cut positions per dimension, and a row-major walk
// over the cells of the resulting grid (last dimension fastest).
using Cuts = std::vector<std::vector<int64_t>>;
void for_each_grid_cell(const Cuts& cuts, const std::function<void(const SliceRegion&)>& fn);

}  // namespace hshard::detail
