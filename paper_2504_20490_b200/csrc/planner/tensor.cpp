// hshard-b200: host Tensor (the reference tensor.hpp API; semantics of its
// tensor.cpp:22-156, planner notice in NOTICE: row-major doubles whatever the
// dtype tag, ShapeMismatch on a box outside the tensor or an empty one, cell
// order row-major over the box).  Box copies here move contiguous innermost
// runs located by precomputed row strides, not one cell per callback.
#include <algorithm>
#include <cmath>
#include <sstream>

#include "hshard/tensor.hpp"

namespace hshard {

int64_t shape_numel(const Shape& s) {
  int64_t n = 1;
  for (int64_t d : s) n *= d;
  return n;
}

Tensor::Tensor(Shape s, DType t) : shape(std::move(s)), dtype(t), data(shape_numel(shape), 0.0) {}

Tensor Tensor::zeros(Shape s, DType t) { return Tensor(std::move(s), t); }

Tensor Tensor::filled(Shape s, double v, DType t) {
  Tensor out(std::move(s), t);
  std::fill(out.data.begin(), out.data.end(), v);
  return out;
}

int64_t Tensor::numel() const { return static_cast<int64_t>(data.size()); }

int64_t Tensor::offset_of(const std::vector<int64_t>& idx) const {
  int64_t off = 0;
  for (size_t d = 0; d < shape.size(); ++d) off = off * shape[d] + idx[d];
  return off;
}

void for_each_cell(const SliceRegion& region,
                   const std::function<void(const std::vector<int64_t>&)>& fn) {
  const size_t rank = region.bounds.size();
  std::vector<int64_t> idx(rank);
  for (size_t d = 0; d < rank; ++d) idx[d] = region.bounds[d][0];
  while (true) {
    fn(idx);
    size_t d = rank;
    for (;;) {
      if (d == 0) return;
      --d;
      if (++idx[d] < region.bounds[d][1]) break;
      idx[d] = region.bounds[d][0];
    }
  }
}

namespace {

void check_box(const Tensor& t, const SliceRegion& r) {
  if (static_cast<int>(r.bounds.size()) != t.ndim())
    fail(Errc::ShapeMismatch, "a rank-" + std::to_string(r.bounds.size()) + " box on a rank-" +
                                  std::to_string(t.ndim()) + " tensor");
  for (size_t d = 0; d < r.bounds.size(); ++d) {
    const auto [lo, hi] = r.bounds[d];
    if (lo < 0 || hi > t.shape[d] || lo >= hi)
      fail(Errc::ShapeMismatch, "box " + r.str() + " is empty or leaves the tensor [" + join_ints(t.shape) + "]");
  }
}

void check_payload(const SliceRegion& r, const Tensor& v) {
  if (v.shape != r.extents())
    fail(Errc::ShapeMismatch, "a [" + join_ints(v.shape) + "] payload for box " + r.str());
}

// fn(tensor_offset, box_offset, run_length) for every innermost run of the
// box, in row-major order; rows are located through the tensor's strides.
template <class Fn>
void for_each_run(const Tensor& t, const SliceRegion& r, Fn&& fn) {
  const size_t rank = r.bounds.size();
  if (rank == 0) {
    fn(int64_t{0}, int64_t{0}, int64_t{1});
    return;
  }
  std::vector<int64_t> stride(rank, 1);
  for (size_t d = rank - 1; d > 0; --d) stride[d - 1] = stride[d] * t.shape[d];
  const int64_t run = r.bounds[rank - 1][1] - r.bounds[rank - 1][0];
  int64_t rows = 1;
  for (size_t d = 0; d + 1 < rank; ++d) rows *= r.bounds[d][1] - r.bounds[d][0];
  for (int64_t row = 0; row < rows; ++row) {
    int64_t at = r.bounds[rank - 1][0], rest = row;
    for (size_t d = rank - 1; d-- > 0;) {
      const int64_t ext = r.bounds[d][1] - r.bounds[d][0];
      at += (r.bounds[d][0] + rest % ext) * stride[d];
      rest /= ext;
    }
    fn(at, row * run, run);
  }
}

}  // namespace

Tensor Tensor::slice(const SliceRegion& region) const {
  check_box(*this, region);
  Tensor out(region.extents(), dtype);
  for_each_run(*this, region, [&](int64_t at, int64_t box, int64_t n) {
    std::copy_n(data.begin() + at, n, out.data.begin() + box);
  });
  return out;
}

void Tensor::write_slice(const SliceRegion& region, const Tensor& value) {
  check_box(*this, region);
  check_payload(region, value);
  for_each_run(*this, region, [&](int64_t at, int64_t box, int64_t n) {
    std::copy_n(value.data.begin() + box, n, data.begin() + at);
  });
}

void Tensor::add_slice(const SliceRegion& region, const Tensor& value) {
  check_box(*this, region);
  check_payload(region, value);
  for_each_run(*this, region, [&](int64_t at, int64_t box, int64_t n) {
    for (int64_t i = 0; i < n; ++i) data[at + i] += value.data[box + i];
  });
}

bool Tensor::bit_equal(const Tensor& o) const { return shape == o.shape && data == o.data; }

double Tensor::max_abs_diff(const Tensor& o) const {
  if (shape != o.shape) fail(Errc::ShapeMismatch, "max_abs_diff of [" + join_ints(shape) + "] and [" + join_ints(o.shape) + "]");
  double m = 0;
  for (size_t i = 0; i < data.size(); ++i) m = std::max(m, std::fabs(data[i] - o.data[i]));
  return m;
}

double Tensor::max_rel_diff(const Tensor& o) const {
  if (shape != o.shape) fail(Errc::ShapeMismatch, "max_rel_diff of [" + join_ints(shape) + "] and [" + join_ints(o.shape) + "]");
  double m = 0;
  for (size_t i = 0; i < data.size(); ++i) {
    const double scale = std::max({std::fabs(data[i]), std::fabs(o.data[i]), 1.0});
    m = std::max(m, std::fabs(data[i] - o.data[i]) / scale);
  }
  return m;
}

Tensor& Tensor::operator+=(const Tensor& o) {
  if (shape != o.shape) fail(Errc::ShapeMismatch, "cannot add [" + join_ints(o.shape) + "] into [" + join_ints(shape) + "]");
  std::transform(data.begin(), data.end(), o.data.begin(), data.begin(), std::plus<double>());
  return *this;
}

std::string Tensor::str() const {
  std::ostringstream os;
  os << dtype_name(dtype) << "[" << join_ints(shape) << "]{";
  const size_t shown = std::min<size_t>(data.size(), 16);
  for (size_t i = 0; i < shown; ++i) os << (i ? "," : "") << data[i];
  if (data.size() > shown) os << ",...";
  os << "}";
  return os.str();
}

}  // namespace hshard
